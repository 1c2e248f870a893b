#!/bin/bash
# round-end style check on 4 GPUs: full GPU suite, smoke, bench N=1 / N=2 / N=4 lines,
# ncu --set full of the fused produce-in-place kernel
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r63_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r63_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/r63_bench1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 > gpurun_out/r63_bench2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 4 > gpurun_out/r63_bench4.log 2>&1
timeout 120 python tools/inplace_ncu.py > gpurun_out/r63_inplace_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:xor_send_kernel -s 2 -c 1 \
    -o gpurun_out/r63_prof_xor_send python tools/inplace_ncu.py > gpurun_out/r63_ncu_xor_send.log 2>&1
true
