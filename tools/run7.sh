timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571 tools/tune_step.py --out gpurun_out/r7_tune.jsonl > gpurun_out/r7_tune.log 2>&1
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "two and (xor or sendrecv)" > gpurun_out/r7_tests.log 2>&1; echo rc=$? >> gpurun_out/r7_tests.log
true
