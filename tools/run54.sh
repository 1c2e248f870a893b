#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_local.py -x -q -k "host or xor_1f1b or graph" > gpurun_out/r54_local.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "host or xor or graph or zero_copy" > gpurun_out/r54_multi.log 2>&1
timeout 300 python bench.py --steps 10 > gpurun_out/r54_bench1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 --steps 10 > gpurun_out/r54_bench2.log 2>&1
true
