#!/bin/bash
# produce-in-place sends with PDL on the header / flags / fused kernels: parity + A/B timing
timeout 600 python -m pytest tests/test_gpu_local.py -x -q -k "produce_in_place or send_recv or xor_1f1b" > gpurun_out/r60_local.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "produce_in_place or two_gpus" > gpurun_out/r60_multi.log 2>&1
for ch in 262144 131072 524288; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 \
  tools/inplace_bench.py --chunk $ch >> gpurun_out/r60_inplace.jsonl 2>> gpurun_out/r60_inplace.err
done
true
