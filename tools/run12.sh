timeout 900 python -m pytest tests/test_gpu_local.py -x -q -k "graph or xor_1f1b" > gpurun_out/r12_tests_local.log 2>&1; echo rc=$? >> gpurun_out/r12_tests_local.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "graph or zero_copy" > gpurun_out/r12_tests_multi.log 2>&1; echo rc=$? >> gpurun_out/r12_tests_multi.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r12_bench1_graph.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --graph 0 > gpurun_out/r12_bench1_eager.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29621 bench.py --gpus 2 > gpurun_out/r12_bench2_graph.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus 2 --graph 0 > gpurun_out/r12_bench2_eager.log 2>&1
true
