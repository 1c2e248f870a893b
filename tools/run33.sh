#!/bin/bash
# PDL on/off, N=1 single transfer queue on/off, N=2 graph; then GPU tests
out=gpurun_out/r33_bench.jsonl; : > $out
for q in 1 0; do for pdl in 1 0; do
  PPC_LOCAL_QUEUE=$q PPC_PDL=$pdl timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>gpurun_out/r33_n1_err.txt | grep '^{' | sed "s/^/{\"n\":1,\"q\":$q,\"pdl\":$pdl,\"line\":/; s/\$/}/" >> $out
done; done
for pdl in 1 0; do
  PPC_PDL=$pdl timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 \
    bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{' | sed "s/^/{\"n\":2,\"pdl\":$pdl,\"line\":/; s/\$/}/" >> $out
done
timeout 900 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/r33_local.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "not gather and not dcbs and not hetero" > gpurun_out/r33_multi.log 2>&1
true
