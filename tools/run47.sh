#!/bin/bash
# bidirectional zero-copy stream: which configurations time out
p() { timeout 60 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29771 tools/zc_bidir.py "$@" 2>&1 | grep "^rank" >> gpurun_out/r47_zc_bidir.log; }
: > gpurun_out/r47_zc_bidir.log
p 64 8
p 128 8
PPC_PDL=0 p 128 8
p 96 8
p 128 2
p 128 3
p 128 4
PPC_PDL=0 p 256 8 128
p 256 8 128
true
