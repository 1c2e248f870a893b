#!/bin/bash
# exposure A/B: stage compute's last GEMM stores into a local buffer + send, or straight into
# the receiver's slot (PPC_STEP_INPLACE); 3 alternating repeats
timeout 300 python -m pytest tests/test_gpu_local.py -x -q -k "produce_in_place" > gpurun_out/r62_local.log 2>&1
for rep in 1 2 3; do
for ip in "" "--inplace"; do
for L in 1 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 \
  bench_exposure.py --layers $L $ip --out gpurun_out/r62_exposure.jsonl > /dev/null 2>> gpurun_out/r62_exposure.err
done; done; done
true
