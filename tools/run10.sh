nvidia-smi topo -m > gpurun_out/r10_topo.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "four or dcbs" > gpurun_out/r10_tests4.log 2>&1; echo rc=$? >> gpurun_out/r10_tests4.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601 bench.py --gpus 4 > gpurun_out/r10_bench4.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 4 --pp 4 --M 16 --no-e2e > gpurun_out/r10_bench4_pp4_m16.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29603 bench.py --gpus 4 --pp 4 --M 32 --hidden 3584 --no-e2e > gpurun_out/r10_bench4_pp4_m32_qwen.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29604 bench.py --gpus 2 > gpurun_out/r10_bench2.log 2>&1
timeout 300 python bench.py > gpurun_out/r10_bench1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29605 bench_stability.py --steps 500 --out gpurun_out/r10_stability2.json > gpurun_out/r10_stability2.log 2>&1
timeout 600 python bench_stability.py --steps 500 --out gpurun_out/r10_stability1.json > gpurun_out/r10_stability1.log 2>&1
true
