#!/bin/bash
: > gpurun_out/r48_zc_bidir.log
p() { timeout 60 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 tools/zc_bidir.py "$@" 2>&1 | grep "^rank" >> gpurun_out/r48_zc_bidir.log; }
p 64 8
p 128 8
p 256 8 128
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r48_multi.log 2>&1
out=gpurun_out/r48_bench.jsonl; : > $out
for rep in 1 2; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus 2 --no-e2e --no-cpu-baseline 2>>gpurun_out/r48_err.txt | grep '^{' | sed "s/^/{\"tag\":\"n2\",\"line\":/; s/\$/}/" >> $out
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
  bench_sweep.py --out gpurun_out/r48_sweep.jsonl --sm 64:512K --ce 1 --zc 64:256K,64:1M \
  --sizes 64K,1M,16M,32M,64M,128M,256M,1G --comparators nccl,ce_copy > gpurun_out/r48_sweep.log 2>&1
true
