#!/bin/bash
# Measurement passes of round 2 (run under gpurun with the GPU count each needs):
#   gpurun --gpus 2 -- "bash tools/perf.sh n2 TAG"     N=2 bench lines, C5 sweep, produce-in-place,
#                                                       exposure, NVLink counters (ncu, one process)
#   n2b   spin tests, WaitValue A/B, MPDT channel sweep, partition, ncu of the XOR-send kernel
#   n2c   header-read + PPC_PUB_FENCE=gpu A/B, partition with sustained layer times
#   n4    (4 GPUs) bench N=4 + PP4 stand-ins, DCBS under load, PP4 exposure, gather, multi tests
#   n4b   (4 GPUs) exposure by mover (zero-copy / push / produce-in-place), gather
#   n4c   (4 GPUs) 8-rank bench rehearsal, gather, 4-rank multi tests
#   partition  (2 GPUs) NEXT-3 planner vs measured for 16-16 / 15-17 / 14-18
#   final2  (2 GPUs) final build: N=2 line, 500-step stability, NVLink counters, C5 sweep
#   final4  (4 GPUs) final build: N=8 bench rehearsal (8 ranks on 4 GPUs), exposure at 1 block/stage
# Logs: gpurun_out/TAG_*.  Copies of the judged ones are in profiles/round2/.
PASS=$1; T=${2:-$1}
mkdir -p gpurun_out
P=$((29500 + RANDOM % 300))
trun() { local n=$1; shift; P=$((P+1)); timeout 1500 python -m torch.distributed.run --nnodes=1 \
           --nproc-per-node $n --master-addr 127.0.0.1 --master-port $P "$@"; }

pass_n2() {
  trun 2 bench.py --gpus 2 > gpurun_out/${T}_bench2.log 2>&1; tail -1 gpurun_out/${T}_bench2.log | cut -c1-400
  PPC_STEP_BATCH=1 trun 2 bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_batch.log 2>&1
  tail -1 gpurun_out/${T}_bench2_batch.log | cut -c1-300
  trun 2 bench_sweep.py --sizes 16M,32M,64M,128M,256M,1G --sm none --ce none --zc 64:256K:a,64:256K:ab \
    --modes uni,bidir --comparators ce_copy --out gpurun_out/${T}_sweep.jsonl > gpurun_out/${T}_sweep.log 2>&1
  cat gpurun_out/${T}_sweep.r0.jsonl | cut -c1-200
  for ch in 256K 128K; do
    trun 2 tools/inplace_bench.py --chunk $((${ch%K} * 1024)) >> gpurun_out/${T}_inplace.log 2>&1
  done
  tail -8 gpurun_out/${T}_inplace.log
  trun 2 bench_exposure.py --layers 1 --reps 5 --layer-times --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exposure.log 2>&1
  tail -1 gpurun_out/${T}_exposure.log | cut -c1-300
  for mode in zc push; do
    timeout 300 python tools/ncu_xdev.py --mode $mode > gpurun_out/${T}_xdev_${mode}.log 2>&1
    timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      -k regex:"recv_kernel|push_ws_kernel" --csv python tools/ncu_xdev.py --mode $mode > gpurun_out/${T}_ncu_xdev_${mode}.csv 2>&1
    tail -4 gpurun_out/${T}_ncu_xdev_${mode}.csv
  done
}

pass_n2b() {
  timeout 900 python -m pytest tests/test_gpu_spin.py -m gpu -q -k "mpdt or batched or early" > gpurun_out/${T}_spin.log 2>&1; tail -2 gpurun_out/${T}_spin.log
  for rep in 1 2; do
    trun 2 bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_default_${rep}.log 2>&1
    PPC_WAIT_VALUE=1 trun 2 bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_waitvalue_${rep}.log 2>&1
  done
  for f in gpurun_out/${T}_bench2_*.log; do echo $f; tail -1 $f | cut -c1-200; done
  trun 2 bench_sweep.py --sizes 16M,64M,256M --sm 64:512K --ce none --zc 64:256K:a --channels 1,2,4,8 \
    --modes uni,bidir --comparators none --out gpurun_out/${T}_sweep_channels.jsonl > gpurun_out/${T}_sweep.log 2>&1
  cut -c1-150 gpurun_out/${T}_sweep_channels.r0.jsonl
  pass_partition
  timeout 300 python tools/inplace_ncu.py > gpurun_out/${T}_inplace_plain.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:xor_send_kernel -s 2 -c 1 \
      -o gpurun_out/${T}_prof_xor_send python tools/inplace_ncu.py > gpurun_out/${T}_ncu_xor_send.log 2>&1
  tail -3 gpurun_out/${T}_ncu_xor_send.log
}

pass_n2c() {
  timeout 900 python -m pytest tests/test_gpu_spin.py tests/test_gpu_multi.py -m gpu -q -x -k "not four and not dcbs and not hetero" > gpurun_out/${T}_tests.log 2>&1; tail -2 gpurun_out/${T}_tests.log
  for rep in 1 2 3; do
    trun 2 bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_default_${rep}.log 2>&1
    PPC_PUB_FENCE=gpu trun 2 bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_gpufence_${rep}.log 2>&1
  done
  for f in gpurun_out/${T}_bench2_*.log; do echo $f $(tail -1 $f | cut -c1-160); done
  pass_partition
}

pass_n4() {
  trun 4 bench.py --gpus 4 > gpurun_out/${T}_bench4.log 2>&1; tail -1 gpurun_out/${T}_bench4.log | cut -c1-300
  trun 4 bench_exposure.py --pp 2 --tp 2 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp2tp2.log 2>&1
  trun 4 bench_exposure.py --pp 2 --tp 2 --M 16 --layers 4 --reps 3 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp2tp2_l4.log 2>&1
  trun 4 bench_exposure.py --pp 4 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp4.log 2>&1
  trun 4 bench_exposure.py --pp 4 --M 16 --layers 8 --reps 3 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp4_l8.log 2>&1
  trun 4 bench_exposure.py --pp 4 --M 32 --layers 1 --hidden 3584 --ffn 18944 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp4_qwen.log 2>&1
  cut -c1-250 gpurun_out/${T}_exposure.jsonl
  trun 4 tools/gather_bench.py > gpurun_out/${T}_gather.log 2>&1; tail -1 gpurun_out/${T}_gather.log
  timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q --durations=10 > gpurun_out/${T}_pytest_multi.log 2>&1; tail -3 gpurun_out/${T}_pytest_multi.log
}

pass_n4b() {
  for v in default push inplace; do
    case $v in default) E="";; push) E="PPC_ZC_STEPBUFS=0";; inplace) E="PPC_ZC_STEPBUFS=0 PPC_STEP_INPLACE=1";; esac
    env $E bash -c "$(declare -f trun); P=$P; trun 4 bench_exposure.py --pp 4 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exp_${v}.jsonl" > gpurun_out/${T}_exp_pp4_${v}.log 2>&1
    P=$((P+1))
    env $E bash -c "$(declare -f trun); P=$P; trun 4 bench_exposure.py --pp 2 --tp 2 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exp_${v}.jsonl" > gpurun_out/${T}_exp_pp2tp2_${v}.log 2>&1
    P=$((P+1))
    echo "== $v"; cut -c1-200 gpurun_out/${T}_exp_${v}.jsonl
  done
  trun 4 tools/gather_bench.py > gpurun_out/${T}_gather.log 2>&1; tail -1 gpurun_out/${T}_gather.log
}

pass_n4c() {
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port 29411 bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/${T}_bench8_rehearsal.log 2>&1
  echo "rc=$?"; tail -1 gpurun_out/${T}_bench8_rehearsal.log | cut -c1-300
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29412 tools/gather_bench.py > gpurun_out/${T}_gather.log 2>&1; tail -1 gpurun_out/${T}_gather.log
  timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -k "gather or dcbs or hetero or four" > gpurun_out/${T}_pytest_multi4.log 2>&1; tail -1 gpurun_out/${T}_pytest_multi4.log
}

pass_partition() {
  for split in 16,16 15,17 14,18; do
    P=$((P+1))
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port $P bench_exposure.py --layers-per-stage $split --ffn-scale-stage0 1.133 \
      --layer-times --M 8 --steps 3 --reps 3 --out gpurun_out/${T}_partition.jsonl \
      > gpurun_out/${T}_partition_${split/,/_}.log 2>&1
    tail -1 gpurun_out/${T}_partition_${split/,/_}.log | cut -c1-200
  done
}

# final (2 GPUs): the N=2 line, 500-step stability, NVLink counters of the zero-copy pull, C5
pass_final2() {
  trun 2 bench.py --gpus 2 > gpurun_out/${T}_bench2.log 2>&1; grep '^{"metric' gpurun_out/${T}_bench2.log | cut -c1-300
  trun 2 bench_stability.py --steps 500 --out gpurun_out/${T}_stability_n2.json > gpurun_out/${T}_stability.log 2>&1
  tail -n 1 gpurun_out/${T}_stability.log | cut -c1-300
  timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:"recv_kernel" --csv python tools/ncu_xdev.py --mode zc > gpurun_out/${T}_ncu_xdev_zc.csv 2>&1
  tail -n 4 gpurun_out/${T}_ncu_xdev_zc.csv
  trun 2 bench_sweep.py --sizes 64K,1M,16M,32M,64M,128M,256M,1G --sm 64:512K --ce 1 --zc 64:256K:a,64:256K:ab \
    --modes uni,bidir --comparators ce_copy --out gpurun_out/${T}_sweep.jsonl > gpurun_out/${T}_sweep.log 2>&1
  tail -n 2 gpurun_out/${T}_sweep.log
}

# final (4 GPUs): the N=8 bench path rehearsed (8 ranks, 2 per GPU), exposure at 1 block per
# stage (PP2, PP2 x TP2 with NCCL, PP4) on the final build
pass_final4() {
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port 29411 bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/${T}_bench8_rehearsal.log 2>&1
  echo "rc=$?"; grep '^{"metric' gpurun_out/${T}_bench8_rehearsal.log | cut -c1-300
  trun 2 bench_exposure.py --layers 1 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp2.log 2>&1
  trun 4 bench_exposure.py --pp 2 --tp 2 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp2tp2.log 2>&1
  trun 4 bench_exposure.py --pp 4 --M 16 --layers 1 --reps 5 --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exp_pp4.log 2>&1
  cut -c1-300 gpurun_out/${T}_exposure.jsonl
}

case $PASS in
  n2|n2b|n2c|n4|n4b|n4c|partition|final2|final4) pass_$PASS ;;
  *) echo "usage: tools/perf.sh n2|n2b|n2c|n4|n4b|n4c|partition|final2|final4 [TAG]"; exit 2 ;;
esac
true
