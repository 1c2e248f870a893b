#!/bin/bash
# fused produce-in-place kernel with 4 input loads in flight per thread: parity, A/B timing,
# ncu --set full
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_local.py -x -q -k "produce_in_place or xor" > gpurun_out/r66_local.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "produce_in_place" > gpurun_out/r66_multi.log 2>&1
for rep in 0 1; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 \
  tools/inplace_bench.py --chunk 262144 >> gpurun_out/r66_inplace.jsonl 2>> gpurun_out/r66_inplace.err
done
timeout 120 python tools/inplace_ncu.py > gpurun_out/r66_inplace_plain.log 2>&1 && \
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:xor_send_kernel -s 2 -c 1 \
    -o gpurun_out/r66_prof_xor_send python tools/inplace_ncu.py > gpurun_out/r66_ncu_xor_send.log 2>&1
true
