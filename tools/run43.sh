#!/bin/bash
# C5 sweep refresh (2 GPUs): zero-copy pulls, SM push, CE; NCCL + CE peer-copy comparators
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
  bench_sweep.py --out gpurun_out/r43_sweep.jsonl --sm 64:512K --ce 1,2 --zc 64:256K,128:256K,64:1M,148:1M \
  --sizes 64K,1M,4M,16M,32M,64M,128M,256M,1G --comparators nccl,ce_copy > gpurun_out/r43_sweep.log 2>&1
true
