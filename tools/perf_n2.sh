#!/bin/bash
# 2-GPU performance pass (run under gpurun --gpus 2): N=2 bench lines (default, batched
# terminal receives), C5 sweep (zero-copy async, +batched receive), produce-in-place A/B,
# exposure with compute, NVLink counters of the cross-GPU kernels (one process, ncu).
T=${1:-p}
mkdir -p gpurun_out
P=29800
trun() { P=$((P+1)); timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
           --master-addr 127.0.0.1 --master-port $P "$@"; }
trun bench.py --gpus 2 > gpurun_out/${T}_bench2.log 2>&1; tail -1 gpurun_out/${T}_bench2.log | cut -c1-400
PPC_STEP_BATCH=1 trun bench.py --gpus 2 --no-b1 --no-e2e > gpurun_out/${T}_bench2_batch.log 2>&1
tail -1 gpurun_out/${T}_bench2_batch.log | cut -c1-300
trun bench_sweep.py --sizes 16M,32M,64M,128M,256M,1G --sm none --ce none --zc 64:256K:a,64:256K:ab \
  --modes uni,bidir --comparators ce_copy --out gpurun_out/${T}_sweep.jsonl > gpurun_out/${T}_sweep.log 2>&1
cat gpurun_out/${T}_sweep.r0.jsonl | cut -c1-200
for ch in 256K 128K; do
  trun tools/inplace_bench.py --chunk $((${ch%K} * 1024)) >> gpurun_out/${T}_inplace.log 2>&1
done
tail -8 gpurun_out/${T}_inplace.log
trun bench_exposure.py --layers 1 --reps 5 --layer-times --out gpurun_out/${T}_exposure.jsonl > gpurun_out/${T}_exposure.log 2>&1
tail -1 gpurun_out/${T}_exposure.log | cut -c1-300
for mode in zc push; do
  timeout 300 python tools/ncu_xdev.py --mode $mode > gpurun_out/${T}_xdev_${mode}.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    -k regex:"recv_kernel|push_ws_kernel" --csv python tools/ncu_xdev.py --mode $mode > gpurun_out/${T}_ncu_xdev_${mode}.csv 2>&1
  tail -4 gpurun_out/${T}_ncu_xdev_${mode}.csv
done
true
