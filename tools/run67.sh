#!/bin/bash
# PPC_RECV_EARLY=1: zero-copy receives look for their publication before griddepcontrol.wait
# and pull their first 64 KiB early.  Parity under the flag, then A/B (N=2 bench, C5 uni/bidir)
mkdir -p gpurun_out
PPC_RECV_EARLY=1 timeout 420 python -m pytest tests/test_gpu_multi.py -x -q -k "two_gpus or zero_copy or cuda_graph or full_size" > gpurun_out/r67_multi_early.log 2>&1
PPC_RECV_EARLY=1 timeout 300 python -m pytest tests/test_gpu_local.py -x -q -k "zero_copy or zc or xor" > gpurun_out/r67_local_early.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 20"
for rep in 0 1 2; do
  for e in 0 1; do
    line=$(PPC_RECV_EARLY=$e timeout 200 $R 2>>gpurun_out/r67_bench.err | grep '^{' | tail -n1)
    echo "{\"early\": $e, \"rep\": $rep, \"line\": ${line:-null}}" >> gpurun_out/r67_n2_early.jsonl
  done
done
for e in 0 1; do
  PPC_RECV_EARLY=$e timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29672 \
    bench_sweep.py --out gpurun_out/r67_sweep_early$e.jsonl --sm "" --ce "" --zc 64:256K,64:64K:a \
    --sizes 32M,64M,128M,256M --comparators "" --reps 3 > gpurun_out/r67_sweep_early$e.log 2>&1
done
true
