#!/bin/bash
# 4-GPU pass (gpurun --gpus 4): bench N=4 (2 x C2 + the PP4 stand-ins of C3 / C4), DCBS under
# load (PP2 x TP2 with NCCL TP allreduces inside the stage compute), PP4 exposure with
# compute (M16, M32 Qwen), TP-sliced gather throughput, the 4-rank GPU tests.
T=${1:-q}
mkdir -p gpurun_out
P=29900
trun() { P=$((P+1)); timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
           --master-addr 127.0.0.1 --master-port $P "$@"; }
trun bench.py --gpus 4 > gpurun_out/${T}_bench4.log 2>&1; tail -1 gpurun_out/${T}_bench4.log | cut -c1-300
trun bench_exposure.py --pp 2 --tp 2 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp2tp2.log 2>&1
trun bench_exposure.py --pp 2 --tp 2 --M 16 --layers 4 --reps 3 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp2tp2_l4.log 2>&1
trun bench_exposure.py --pp 4 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp4.log 2>&1
trun bench_exposure.py --pp 4 --M 16 --layers 8 --reps 3 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp4_l8.log 2>&1
trun bench_exposure.py --pp 4 --M 32 --layers 1 --hidden 3584 --ffn 18944 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp4_qwen.log 2>&1
cut -c1-250 gpurun_out/${T}_exposure.jsonl
trun tools/gather_bench.py > gpurun_out/${T}_gather.log 2>&1; tail -1 gpurun_out/${T}_gather.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q --durations=10 > gpurun_out/${T}_pytest_multi.log 2>&1; tail -3 gpurun_out/${T}_pytest_multi.log
true
