#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "zero_copy" > gpurun_out/r49_multi.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
  bench_sweep.py --out gpurun_out/r49_sweep.jsonl --sm "" --ce "" --zc 64:256K,64:256K:a,64:1M:a \
  --sizes 1M,16M,32M,64M,128M,256M,1G --comparators "" > gpurun_out/r49_sweep.log 2>&1
true
