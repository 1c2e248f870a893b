#!/bin/bash
# final round-end style check of the committed build (defaults): GPU suite on 2 GPUs, smoke, N=1 bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q > gpurun_out/r68_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r68_smoke.log 2>&1
timeout 300 python bench.py > gpurun_out/r68_bench1.log 2>&1
true
