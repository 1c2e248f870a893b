#!/bin/bash
# zero-copy publication on the send stream (PPC_ZC_SIDE=1, new default) vs the compute stream
: > gpurun_out/r32_bench.jsonl
for side in 1 0; do for g in 1 0; do
  PPC_ZC_SIDE=$side timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 \
    bench.py --gpus 2 --steps 30 --warmup 5 --graph $g --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | sed "s/^/{\"side\":$side,\"g\":$g,\"line\":/; s/\$/}/" >> gpurun_out/r32_bench.jsonl
done; done
for g in 0 1; do
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 tools/timeline.py --zc 1 --chunk 262144 --graph $g > gpurun_out/r32_tl_g$g.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "zc or graph or fullsize or toy" > gpurun_out/r32_multi.log 2>&1
true
