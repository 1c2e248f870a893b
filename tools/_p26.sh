mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_spin.py -q -x > gpurun_out/p26_spin.log 2>&1; tail -n 2 gpurun_out/p26_spin.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x > gpurun_out/p26_multi.log 2>&1; tail -n 2 gpurun_out/p26_multi.log
P=29500
for r in 1 2 3; do
  for cfg in "0 0" "1 0" "0 1" "1 1"; do
    set -- $cfg; P=$((P+1))
    PPC_RECV_CHAIN=$1 PPC_PUB_BLOCK0=$2 timeout 300 $B --master-port $P bench.py --gpus 2 --no-e2e --no-cpu-baseline --no-b1 --no-extra > gpurun_out/p26_bench2_c$1_b$2_$r.log 2>&1
    echo "chain=$1 b0=$2 $(grep '^{"metric' gpurun_out/p26_bench2_c$1_b$2_$r.log | cut -c1-260)"
  done
done
P=$((P+1)); PPC_DBG_STAMPS=1 timeout 300 $B --master-port $P tools/hop_stamps.py --graph > gpurun_out/p26_hop_graph.log 2>&1; tail -n 1 gpurun_out/p26_hop_graph.log | cut -c1-700
cp gpurun_out/hop_stamps.json gpurun_out/p26_hop_stamps_graph.json 2>/dev/null
