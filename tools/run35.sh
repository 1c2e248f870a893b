#!/bin/bash
# N=2 engines with graph + PDL (C2 PP2 M8)
out=gpurun_out/r35_bench.jsonl; : > $out
run() {  # tag args...
  tag=$1; shift
  timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 \
    bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline "$@" 2>>gpurun_out/r35_err.txt | grep '^{' | sed "s/^/{\"tag\":\"$tag\",\"line\":/; s/\$/}/" >> $out
}
run zc --zc 1
run ring_sm --zc 0
run ring_sm_c1m --zc 0 --chunk 1048576
run ring_ce --zc 0 --engine ce
run ring_ce_ch2 --zc 0 --engine ce --channels 2
run ring_pull --zc 0 --engine pull
run zc_c512k --zc 1 --chunk 524288
run zc_c128k --zc 1 --chunk 131072
PPC_RECV_CTAS=96 run zc_r96 --zc 1
PPC_RECV_CTAS=128 run zc_r128 --zc 1
PPC_RECV_CTAS=48 run zc_r48 --zc 1
true
