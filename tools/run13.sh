timeout 900 python -m pytest tests/test_gpu_local.py -x -q -k "graph" > gpurun_out/r13_tests_local.log 2>&1; echo rc=$? >> gpurun_out/r13_tests_local.log
PPC_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "graph" > gpurun_out/r13_tests_multi.log 2>&1; echo rc=$? >> gpurun_out/r13_tests_multi.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 2 > gpurun_out/r13_bench2_graph.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench_sweep.py --out gpurun_out/r13_sweep.jsonl --sm 64:512K,128:256K --ce 1,2 --pull 64:256K --zc 64:256K,128:256K --sizes 64K,1M,4M,16M,28M,32M,64M,256M,1G > gpurun_out/r13_sweep.log 2>&1
true
