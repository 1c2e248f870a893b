#!/bin/bash
# (1) PP4: middle-stage zero-copy forwarding from arena step buffers on/off (ring sources)
# (2) N=2 C2: receive CTAs x chunk, 3 repeats
out=gpurun_out/r40_bench.jsonl; : > $out
run() {
  tag=$1; n=$2; shift; shift
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29781 \
    bench.py --gpus $n --no-e2e --no-cpu-baseline "$@" 2>>gpurun_out/r40_err.txt | grep '^{' | sed "s/^/{\"tag\":\"$tag\",\"line\":/; s/\$/}/" >> $out
}
for rep in 1 2; do
  PPC_ZC_STEPBUFS=1 run pp4m16_step1 4 --pp 4 --M 16 --zc 0
  PPC_ZC_STEPBUFS=0 run pp4m16_step0 4 --pp 4 --M 16 --zc 0
done
for rep in 1 2 3; do
  for r in 64 96 128 148; do
    PPC_RECV_CTAS=$r run n2_r${r}_c256 2 --zc 1 --chunk 262144
  done
  PPC_RECV_CTAS=128 run n2_r128_c512 2 --zc 1 --chunk 524288
  PPC_RECV_CTAS=128 run n2_r128_c128 2 --zc 1 --chunk 131072
done
true
