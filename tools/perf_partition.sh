#!/bin/bash
# NEXT-3 on 2 GPUs: the partition planner fed with measured per-layer times.  Stage 0 is made
# 13.3 % slower per layer (ffn x 1.133, the paper's AMD:NVIDIA ratio in SPEC S:L557); the
# LLaMA-8B 32 MLP blocks are split 16-16 (even), then as the planner recommends, then one
# further; each run prints the planner's predicted step time beside the measured one.
T=${1:-part}
mkdir -p gpurun_out
P=29950
for split in 16,16 15,17 14,18; do
  P=$((P+1))
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $P bench_exposure.py --layers-per-stage $split --ffn-scale-stage0 1.133 \
    --layer-times --M 8 --steps 3 --reps 3 --out gpurun_out/${T}_partition.jsonl \
    > gpurun_out/${T}_partition_${split/,/_}.log 2>&1
  tail -1 gpurun_out/${T}_partition_${split/,/_}.log | cut -c1-200
done
true
