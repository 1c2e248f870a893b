#!/bin/bash
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 > gpurun_out/r53_bench2.log 2>&1
timeout 300 python bench.py > gpurun_out/r53_bench1.log 2>&1
true
