#!/bin/bash
# round measurements on 4 GPUs: N=2/N=4 bench lines, PP4 stand-ins, stability, exposure, reference arm
tr() { n=$1; port=$2; shift; shift; timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port "$@"; }
tr 2 29701 bench.py --gpus 2 > gpurun_out/r44_bench2.log 2>&1
tr 4 29702 bench.py --gpus 4 > gpurun_out/r44_bench4.log 2>&1
tr 4 29703 bench.py --gpus 4 --pp 4 --M 16 --no-e2e > gpurun_out/r44_bench4_pp4_m16.log 2>&1
tr 4 29704 bench.py --gpus 4 --pp 4 --M 32 --hidden 3584 --no-e2e > gpurun_out/r44_bench4_pp4_m32_qwen.log 2>&1
tr 2 29705 bench.py --gpus 2 --impl reference --steps 3 --warmup 1 > gpurun_out/r44_reference2.log 2>&1
tr 2 29706 bench_stability.py --steps 500 --out gpurun_out/r44_stability_n2.json > gpurun_out/r44_stability_n2.log 2>&1
timeout 300 python bench_stability.py --steps 500 --out gpurun_out/r44_stability_n1.json > gpurun_out/r44_stability_n1.log 2>&1
tr 2 29707 bench_exposure.py --layers 1 > gpurun_out/r44_exposure_l1.log 2>&1
tr 2 29708 bench_exposure.py --layers 4 > gpurun_out/r44_exposure_l4.log 2>&1
true
