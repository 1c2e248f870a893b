timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "graph or zero_copy or xor" > gpurun_out/r18_tests.log 2>&1; echo rc=$? >> gpurun_out/r18_tests.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29681 bench.py --gpus 2 > gpurun_out/r18_bench2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29682 bench.py --gpus 2 --graph 0 --no-e2e > gpurun_out/r18_bench2_eager.log 2>&1
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29683 tools/timeline.py --zc 1 --chunk 262144 --out gpurun_out/r18_tl > gpurun_out/r18_timeline.log 2>&1
true
