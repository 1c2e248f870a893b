#!/bin/bash
# receive kernel variants (plain 64 regs / fused publication 88 regs), spinning grids clamped to residency
timeout 900 python -m pytest tests/test_gpu_local.py tests/test_gpu_toy.py -x -q > gpurun_out/r46_local.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r46_multi.log 2>&1
out=gpurun_out/r46_bench.jsonl; : > $out
run() {
  tag=$1; n=$2; shift; shift
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus $n --no-e2e --no-cpu-baseline "$@" 2>>gpurun_out/r46_err.txt | grep '^{' | sed "s/^/{\"tag\":\"$tag\",\"line\":/; s/\$/}/" >> $out
}
for rep in 1 2; do run n2 2; done
run pp4m16 4 --pp 4 --M 16
run pp4m32q 4 --pp 4 --M 32 --hidden 3584
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
  bench_sweep.py --out gpurun_out/r46_sweep.jsonl --sm "" --ce "" --zc 64:256K,128:256K,148:256K \
  --sizes 16M,32M,64M,256M --comparators "" --modes bidir,uni > gpurun_out/r46_sweep.log 2>&1
true
