#!/bin/bash
# 4 GPUs: full multi-GPU test file, then PP4 benches with arena zero-copy forwarding
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r38_multi.log 2>&1
out=gpurun_out/r38_bench.jsonl; : > $out
run() {
  tag=$1; shift
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus 4 --no-e2e --no-cpu-baseline "$@" 2>>gpurun_out/r38_err.txt | grep '^{' | sed "s/^/{\"tag\":\"$tag\",\"line\":/; s/\$/}/" >> $out
}
run pp4m16_zc --pp 4 --M 16 --zc 1
run pp4m16_ring --pp 4 --M 16 --zc 0
PPC_ZC_STEPBUFS=0 run pp4m16_zc_nostep --pp 4 --M 16 --zc 1
run pp4m32q_zc --pp 4 --M 32 --hidden 3584 --zc 1
run pp4m32q_ring --pp 4 --M 32 --hidden 3584 --zc 0
run pp2x2 --pp 2
true
