#!/bin/bash
# fused publication (recv kernel publishes the next zero-copy send) on/off
out=gpurun_out/r36_bench.jsonl; : > $out
for f in 1 0; do
  PPC_FUSE_PUBLISH=$f timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 \
    bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/r36_err.txt | grep '^{' | sed "s/^/{\"fuse\":$f,\"line\":/; s/\$/}/" >> $out
  PPC_FUSE_PUBLISH=$f timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 \
    bench.py --gpus 2 --steps 30 --warmup 5 --seq 1 --hidden 8 --no-e2e --no-cpu-baseline 2>>gpurun_out/r36_err.txt | grep '^{' | sed "s/^/{\"fuse\":$f,\"tiny\":1,\"line\":/; s/\$/}/" >> $out
done
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 tools/timeline.py --zc 1 --chunk 262144 --graph 1 > gpurun_out/r36_tl_g1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "not gather and not dcbs and not hetero" > gpurun_out/r36_multi.log 2>&1
timeout 600 python -m pytest tests/test_gpu_local.py tests/test_gpu_toy.py -x -q > gpurun_out/r36_local.log 2>&1
true
