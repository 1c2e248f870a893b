#!/bin/bash
# 4-GPU pass B: exposed PP comm at 1 block per stage — zero-copy forwarding from the step
# buffers (default: the receiver pulls when it reaches its receive) vs ring push (the sender
# pushes as soon as its op ends, PPC_ZC_STEPBUFS=0) vs produce-in-place; gather after the
# sender-interleaved unit order.
T=${1:-qb}
mkdir -p gpurun_out
P=29500
trun() { P=$((P+1)); timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
           --master-addr 127.0.0.1 --master-port $P "$@"; }
for v in default push inplace; do
  case $v in default) E="";; push) E="PPC_ZC_STEPBUFS=0";; inplace) E="PPC_ZC_STEPBUFS=0 PPC_STEP_INPLACE=1";; esac
  env $E bash -c "$(declare -f trun); P=$P; trun bench_exposure.py --pp 4 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exp_${v}.jsonl" > gpurun_out/${T}_exp_pp4_${v}.log 2>&1
  P=$((P+1))
  env $E bash -c "$(declare -f trun); P=$P; trun bench_exposure.py --pp 2 --tp 2 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exp_${v}.jsonl" > gpurun_out/${T}_exp_pp2tp2_${v}.log 2>&1
  P=$((P+1))
  echo "== $v"; cut -c1-200 gpurun_out/${T}_exp_${v}.jsonl
done
trun tools/gather_bench.py > gpurun_out/${T}_gather.log 2>&1; tail -1 gpurun_out/${T}_gather.log
true
