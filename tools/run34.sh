#!/bin/bash
# N=1: single transfer queue on/off x copy grid; predicated grid-stride copy_kernel
out=gpurun_out/r34_bench.jsonl; : > $out
for q in 1 0; do for ctas in 296 148; do
  PPC_LOCAL_QUEUE=$q PPC_COPY_CTAS=$ctas timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>>gpurun_out/r34_err.txt | grep '^{' | sed "s/^/{\"q\":$q,\"ctas\":$ctas,\"line\":/; s/\$/}/" >> $out
done; done
timeout 600 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/r34_local.log 2>&1
true
