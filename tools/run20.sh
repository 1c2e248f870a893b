timeout 900 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/r20_tests_local.log 2>&1; echo rc=$? >> gpurun_out/r20_tests_local.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 4 --pp 4 --M 16 --no-e2e > gpurun_out/r20_bench4_pp4_m16.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29702 bench.py --gpus 4 --pp 4 --M 32 --hidden 3584 --no-e2e > gpurun_out/r20_bench4_pp4_m32_qwen.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29703 bench.py --gpus 4 --pp 4 --M 16 --no-e2e --zc 0 > gpurun_out/r20_bench4_pp4_m16_ring.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29704 bench.py --gpus 2 > gpurun_out/r20_bench2.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/r20_tests_multi.log 2>&1; echo rc=$? >> gpurun_out/r20_tests_multi.log
true
