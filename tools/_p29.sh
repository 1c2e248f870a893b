mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
L=paper_2602_18007_b200/libppc.so
cp ab_tmp/libppc_new.so $L
timeout 900 python -m pytest tests/test_gpu_spin.py -q -x > gpurun_out/p29_spin.log 2>&1; tail -n 2 gpurun_out/p29_spin.log
P=29500
for r in 1 2 3 4; do
  for v in prev new; do
    cp ab_tmp/libppc_$v.so $L; P=$((P+1))
    timeout 300 $B --master-port $P bench.py --gpus 2 --no-e2e --no-cpu-baseline --no-b1 --no-extra > gpurun_out/p29_bench2_${v}_$r.log 2>&1
    echo "$v $(grep '^{"metric' gpurun_out/p29_bench2_${v}_$r.log | cut -c150-200)"
  done
done
cp ab_tmp/libppc_new.so $L
P=$((P+1)); PPC_DBG_STAMPS=1 timeout 300 $B --master-port $P tools/hop_stamps.py --graph > gpurun_out/p29_hop_graph.log 2>&1; tail -n 1 gpurun_out/p29_hop_graph.log | cut -c1-700
cp gpurun_out/hop_stamps.json gpurun_out/p29_hop_stamps_graph.json 2>/dev/null
