set -x
timeout 600 python -m pytest tests/test_gpu_local.py tests/test_gpu_multi.py -x -q -k "not four and not dcbs" > gpurun_out/r5_tests.log 2>&1; echo rc=$? >> gpurun_out/r5_tests.log
for eng in sm pull; do for sz in 32M 256M; do for cta in 32 64 128; do
  timeout 60 python tools/xdev_push.py --size $sz --n 20 --cta $cta --chunk 1M --engine $eng >> gpurun_out/r5_xdev.jsonl 2>>gpurun_out/r5_xdev.err
done; done; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench_sweep.py --out gpurun_out/r5_sweep.jsonl --sm "" --ce "" --pull "32:1M,64:1M,64:256K,128:256K,128:512K" --comparators "" --sizes 1M,4M,16M,32M,64M,256M,1G > gpurun_out/r5_sweep.log 2>&1
for eng in sm pull; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 bench.py --gpus 2 --no-e2e --engine $eng > gpurun_out/r5_bench2_$eng.log 2>&1
done
true
