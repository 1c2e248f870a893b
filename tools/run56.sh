#!/bin/bash
# TMA bulk hand-off copy (K11): parity of the direct path, N=1 bench A/B vs the SIMT copy,
# launch list and ncu --set full of copy_tma_kernel
timeout 900 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/r56_local.log 2>&1
for c in 148 296 0 148; do
  PPC_COPY_TMA_CTAS=$c timeout 300 python bench.py --steps 20 --no-e2e --no-cpu-baseline > gpurun_out/r56_bench1_tma$c.log 2>&1
done
timeout 300 python bench.py > gpurun_out/r56_bench1.log 2>&1
timeout 120 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r56_plain.log 2>&1 && \
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r56_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r56_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_tma_kernel -s 40 -c 2 \
    -o gpurun_out/r56_prof_copy_tma python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r56_ncu_copy.log 2>&1
true
