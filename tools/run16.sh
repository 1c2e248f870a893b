python tools/graph_debug.py > gpurun_out/r16_gdbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_local.py -x -q -k "graph" > gpurun_out/r16_tests_local.log 2>&1; echo rc=$? >> gpurun_out/r16_tests_local.log
PPC_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "graph" > gpurun_out/r16_tests_multi.log 2>&1; echo rc=$? >> gpurun_out/r16_tests_multi.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r16_bench1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 2 > gpurun_out/r16_bench2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 2 --zc 0 > gpurun_out/r16_bench2_ring.log 2>&1
true
