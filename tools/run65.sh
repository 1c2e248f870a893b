#!/bin/bash
# N=2 C2 step: copy-engine ring sends (CE+CE is the fastest bidirectional mover in
# profiles/r29_nvlink_bidir.md) vs the default zero-copy pull, same box, 2 repeats
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 2 --no-e2e --no-cpu-baseline --steps 20"
for rep in 0 1; do
  for cfg in "zc::" "ce_ch1:--engine ce --zc 0 --channels 1" "ce_ch2:--engine ce --zc 0 --channels 2" \
             "ce_ch4:--engine ce --zc 0 --channels 4" "ce_ch1_k4:--engine ce --zc 0 --slots 4" \
             "ring_sm:--engine sm --zc 0"; do
    tag=${cfg%%:*}; args=${cfg#*:}
    line=$(timeout 200 $R $args 2>gpurun_out/r65_${tag}_${rep}.err | grep '^{' | tail -n1)
    echo "{\"tag\": \"$tag\", \"rep\": $rep, \"line\": ${line:-null}}" >> gpurun_out/r65_n2_ce.jsonl
  done
done
true
