#!/bin/bash
# 4-GPU pass C: the 8-rank bench path rehearsed on 4 GPUs (2 ranks per GPU: correctness of
# the N=8 code path incl. the C3 / C4 extras, not a measurement), TP-sliced gather after the
# side-stream credit, the 4-rank GPU tests.
T=${1:-qc}
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
  --master-port 29411 bench.py --gpus 8 --steps 5 --warmup 3 > gpurun_out/${T}_bench8_rehearsal.log 2>&1
echo "rc=$?"; tail -1 gpurun_out/${T}_bench8_rehearsal.log | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29412 tools/gather_bench.py > gpurun_out/${T}_gather.log 2>&1; tail -1 gpurun_out/${T}_gather.log
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q -k "gather or dcbs or hetero or four" > gpurun_out/${T}_pytest_multi4.log 2>&1; tail -1 gpurun_out/${T}_pytest_multi4.log
true
