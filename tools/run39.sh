#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_local.py tests/test_gpu_toy.py -x -q > gpurun_out/r39_local.log 2>&1
timeout 300 python bench.py > gpurun_out/r39_bench1.log 2>&1
timeout 120 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r39_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r39_launches_n1.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r39_ncu_launch.log 2>&1
true
