mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 > gpurun_out/q41_bench4.log 2>&1; grep '^{"metric' gpurun_out/q41_bench4.log | cut -c1-200
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 > gpurun_out/q41_bench2.log 2>&1; grep '^{"metric' gpurun_out/q41_bench2.log | cut -c1-200
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/q41_tests.log 2>&1; tail -n 2 gpurun_out/q41_tests.log
