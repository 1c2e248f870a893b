#!/bin/bash
# single fence + relaxed flag and credit stores: tests + N=2 bench x3 + timeline
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "zero_copy or graph or full_size or xor or toy" > gpurun_out/r42_multi.log 2>&1
out=gpurun_out/r42_bench.jsonl; : > $out
for rep in 1 2 3; do
  timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 \
    bench.py --gpus 2 --no-e2e --no-cpu-baseline 2>>gpurun_out/r42_err.txt | grep '^{' | sed "s/^/{\"tag\":\"relaxed\",\"line\":/; s/\$/}/" >> $out
done
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 tools/timeline.py --zc 1 --chunk 262144 --graph 1 > gpurun_out/r42_tl_g1.txt 2>&1
true
