#!/bin/bash
# occupancy-gated PDL, fused-publication registers: 4-GPU tests, N=2 / PP4 regression, bidir zc sweep
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r45_multi.log 2>&1
out=gpurun_out/r45_bench.jsonl; : > $out
run() {
  tag=$1; n=$2; shift; shift
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus $n --no-e2e --no-cpu-baseline "$@" 2>>gpurun_out/r45_err.txt | grep '^{' | sed "s/^/{\"tag\":\"$tag\",\"line\":/; s/\$/}/" >> $out
}
for rep in 1 2; do run n2 2; run pp4m16 4 --pp 4 --M 16; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
  bench_sweep.py --out gpurun_out/r45_sweep.jsonl --sm "" --ce "" --zc 64:256K,128:256K \
  --sizes 16M,32M,64M,256M --comparators "" --modes bidir > gpurun_out/r45_sweep.log 2>&1
true
