#!/bin/bash
# 2-GPU pass C: header-read change + PPC_PUB_FENCE=gpu A/B on the N=2 step (alternating
# repeats), spin tests, partition planner with sustained per-layer times.
T=${1:-pc}
mkdir -p gpurun_out
P=29600
trun() { P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
           --master-addr 127.0.0.1 --master-port $P "$@"; }
timeout 900 python -m pytest tests/test_gpu_spin.py tests/test_gpu_multi.py -m gpu -q -x -k "not four and not dcbs and not hetero" > gpurun_out/${T}_tests.log 2>&1; tail -2 gpurun_out/${T}_tests.log
for rep in 1 2 3; do
  trun bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_default_${rep}.log 2>&1
  PPC_PUB_FENCE=gpu trun bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_gpufence_${rep}.log 2>&1
done
for f in gpurun_out/${T}_bench2_*.log; do echo $f $(tail -1 $f | cut -c1-160); done
bash tools/perf_partition.sh ${T}
true
