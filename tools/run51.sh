#!/bin/bash
# round-end check: the whole GPU test suite + smoke on a 4-GPU box
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r51_pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r51_smoke.log 2>&1
true
