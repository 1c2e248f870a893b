#!/bin/bash
# round-end style check on 2 GPUs: full GPU suite, smoke, bench N=1 / N=2 lines, launch list of
# the N=1 bench, ncu --set full of the fused produce-in-place kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r64_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r64_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/r64_bench1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 > gpurun_out/r64_bench2.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/r64_reference.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r64_launches_n1.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r64_ncu_launches.log 2>&1
timeout 120 python tools/inplace_ncu.py > gpurun_out/r64_inplace_plain.log 2>&1 && \
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:xor_send_kernel -s 2 -c 1 \
    -o gpurun_out/r64_prof_xor_send python tools/inplace_ncu.py > gpurun_out/r64_ncu_xor_send.log 2>&1
true
