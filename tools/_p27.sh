mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
PPC_PULL_DYN=1 timeout 900 python -m pytest tests/test_gpu_spin.py -q -x > gpurun_out/p27_spin_dyn.log 2>&1; tail -n 2 gpurun_out/p27_spin_dyn.log
P=29500
for r in 1 2 3; do
  for dy in 0 1; do
    P=$((P+1))
    PPC_PULL_DYN=$dy timeout 300 $B --master-port $P bench.py --gpus 2 --no-e2e --no-cpu-baseline --no-b1 --no-extra > gpurun_out/p27_bench2_dyn${dy}_$r.log 2>&1
    echo "dyn=$dy $(grep '^{"metric' gpurun_out/p27_bench2_dyn${dy}_$r.log | cut -c150-200)"
  done
done
P=$((P+1)); PPC_PULL_DYN=1 PPC_DBG_STAMPS=1 timeout 300 $B --master-port $P tools/hop_stamps.py --graph > gpurun_out/p27_hop_graph.log 2>&1; tail -n 1 gpurun_out/p27_hop_graph.log | cut -c1-700
cp gpurun_out/hop_stamps.json gpurun_out/p27_hop_stamps_graph_dyn.json 2>/dev/null
P=$((P+1)); PPC_PULL_DYN=1 timeout 600 $B --master-port $P bench_sweep.py --sizes 32M,64M,256M --sm none --ce none --zc 64:256K:a,64:256K:ab --comparators none --out gpurun_out/p27_c5_dyn.jsonl > gpurun_out/p27_c5.log 2>&1; tail -n 3 gpurun_out/p27_c5.log
