set -x
./tools/nvlink_probe > gpurun_out/r6_probe.jsonl 2> gpurun_out/r6_probe.err
for e in sm pull; do
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/timeline.py --engine $e --out gpurun_out/r6_tl_$e > gpurun_out/r6_timeline_$e.log 2>&1
done
true
