#!/bin/bash
# produce-in-place sends: parity on 1 GPU (virtual stages) and 2 GPUs, then the A/B timing
timeout 600 python -m pytest tests/test_gpu_local.py -x -q -k "produce_in_place or send_recv or misaligned" > gpurun_out/r59_local.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "produce_in_place or two_gpus" > gpurun_out/r59_multi.log 2>&1
for ch in 524288 1048576 262144; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 \
  tools/inplace_bench.py --chunk $ch >> gpurun_out/r59_inplace.jsonl 2>> gpurun_out/r59_inplace.err
done
true
