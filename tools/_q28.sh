mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29600
P=$((P+1)); timeout 600 $B --master-port $P bench.py --gpus 4 > gpurun_out/q28_bench4.log 2>&1; grep '^{"metric' gpurun_out/q28_bench4.log | cut -c1-250
for wl in C3-pp4 C4-pp4; do for zc in 0 1; do
  P=$((P+1)); timeout 400 $B --master-port $P bench.py --gpus 4 --workload $wl --zc $zc --no-e2e --no-cpu-baseline --no-b1 --no-extra > gpurun_out/q28_${wl}_zc$zc.log 2>&1
  echo "$wl zc=$zc $(grep '^{"metric' gpurun_out/q28_${wl}_zc$zc.log | cut -c150-210)"
done; done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/q28_tests.log 2>&1; tail -n 2 gpurun_out/q28_tests.log
