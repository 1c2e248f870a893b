#!/bin/bash
timeout 300 python bench.py > gpurun_out/r50_bench1.log 2>&1
timeout 120 python tools/xdev_push.py --size 32M --n 4 --engine pull --cta 64 --chunk 256K > gpurun_out/r50_plain_xdev.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:recv_kernel -s 6 -c 2 \
    -o gpurun_out/r50_prof_pull python tools/xdev_push.py --size 32M --n 4 --engine pull --cta 64 --chunk 256K > gpurun_out/r50_ncu_pull.log 2>&1
true
