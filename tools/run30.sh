#!/bin/bash
# latency chain of the PP2 step: tiny messages, graph on/off, zero-copy on/off
out=gpurun_out/r30_lat.jsonl; : > $out
for g in 1 0; do for zc in 1 0; do
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 \
    bench.py --gpus 2 --steps 50 --warmup 5 --seq 1 --hidden 8 --graph $g --zc $zc --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | sed "s/^/{\"g\":$g,\"zc\":$zc,\"line\":/; s/\$/}/" >> $out
done; done
