timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "zero_copy or hetero or two" > gpurun_out/r11_tests.log 2>&1; echo rc=$? >> gpurun_out/r11_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/tune_step.py --out gpurun_out/r11_tune.jsonl --sm 524288:64:64 --pull "" > gpurun_out/r11_tune.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 > gpurun_out/r11_bench2.log 2>&1
true
