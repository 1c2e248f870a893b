#!/bin/bash
# zero-copy pull with dynamic chunk assignment: parity (2 GPUs), C5 sweep and N=2 bench A/B
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "zero_copy or xor or graph or host" > gpurun_out/r57_multi.log 2>&1
for dyn in 1 0; do
  PPC_RECV_DYNAMIC=$dyn timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
    bench_sweep.py --out gpurun_out/r57_sweep_dyn$dyn.jsonl --sm "" --ce "" --zc 64:64K:a,64:32K:a,64:128K:a \
    --sizes 32M,64M,128M,256M --modes uni,bidir --comparators "" > gpurun_out/r57_sweep_dyn$dyn.log 2>&1
done
out=gpurun_out/r57_bench2.jsonl; : > $out
for dyn in 1 0 1 0; do
  PPC_RECV_DYNAMIC=$dyn timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus 2 --no-e2e --no-cpu-baseline 2>>gpurun_out/r57_err.txt | grep '^{' | sed "s/^/{\"dyn\":$dyn,\"line\":/; s/\$/}/" >> $out
done
true
