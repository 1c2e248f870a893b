#!/bin/bash
# 2-GPU pass B: spin-mode tests (MPDT channels), N=2 bench A/B of cuStreamWaitValue64 credit
# waits, C5 sweep over MPDT channel counts, partition planner with sustained-clock layer
# times, ncu --set full of the fused XOR-send kernel.
T=${1:-pb}
mkdir -p gpurun_out
P=29700
trun() { P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
           --master-addr 127.0.0.1 --master-port $P "$@"; }
timeout 900 python -m pytest tests/test_gpu_spin.py -m gpu -q -k "mpdt or batched or early" > gpurun_out/${T}_spin.log 2>&1; tail -2 gpurun_out/${T}_spin.log
for rep in 1 2; do
  trun bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_default_${rep}.log 2>&1
  PPC_WAIT_VALUE=1 trun bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_waitvalue_${rep}.log 2>&1
done
for f in gpurun_out/${T}_bench2_*.log; do echo $f; tail -1 $f | cut -c1-200; done
trun bench_sweep.py --sizes 16M,64M,256M --sm 64:512K --ce none --zc 64:256K:a --channels 1,2,4,8 \
  --modes uni,bidir --comparators none --out gpurun_out/${T}_sweep_channels.jsonl > gpurun_out/${T}_sweep.log 2>&1
cut -c1-150 gpurun_out/${T}_sweep_channels.r0.jsonl
bash tools/perf_partition.sh ${T}
timeout 300 python tools/inplace_ncu.py > gpurun_out/${T}_inplace_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:xor_send_kernel -s 2 -c 1 \
    -o gpurun_out/${T}_prof_xor_send python tools/inplace_ncu.py > gpurun_out/${T}_ncu_xor_send.log 2>&1
tail -3 gpurun_out/${T}_ncu_xor_send.log
true
