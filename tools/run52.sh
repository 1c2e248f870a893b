#!/bin/bash
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 \
  bench_sweep.py --out gpurun_out/r52_sweep.jsonl --sm "" --ce "" --zc 64:64K:a,64:128K:a,64:256K:a,64:64K \
  --sizes 32M,64M,128M,256M --modes uni,bidir --comparators "" > gpurun_out/r52_sweep.log 2>&1
out=gpurun_out/r52_bench.jsonl; : > $out
for c in 65536 131072 262144; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus 2 --no-e2e --no-cpu-baseline --chunk $c 2>>gpurun_out/r52_err.txt | grep '^{' | sed "s/^/{\"chunk\":$c,\"line\":/; s/\$/}/" >> $out
done
true
