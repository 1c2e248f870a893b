#!/bin/bash
# round-end style N=1 measurements + ncu --set full of the direct-mode copy kernel
timeout 300 python bench.py > gpurun_out/r37_bench1.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r37_reference.log 2>&1
timeout 120 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r37_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 40 -c 2 \
    -o gpurun_out/r37_prof_copy python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r37_ncu_copy.log 2>&1
true
