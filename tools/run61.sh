#!/bin/bash
# step driver with produce-in-place stage fns: parity (1 and 2 GPUs), exposure A/B with
# LLaMA-MLP stage compute whose last GEMM stores into the receiver's slot
timeout 600 python -m pytest tests/test_gpu_local.py -x -q -k "produce_in_place or xor_1f1b" > gpurun_out/r61_local.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "produce_in_place or xor" > gpurun_out/r61_multi.log 2>&1
for rep in 1 2; do
for ip in "" "--inplace"; do
for L in 1 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 \
  bench_exposure.py --layers $L $ip --out gpurun_out/r61_exposure.jsonl > /dev/null 2>> gpurun_out/r61_exposure.err
done; done; done
true
