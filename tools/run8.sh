timeout 600 python -m pytest tests/test_gpu_local.py tests/test_gpu_multi.py -x -q -k "not four and not dcbs" > gpurun_out/r8_tests.log 2>&1; echo rc=$? >> gpurun_out/r8_tests.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 tools/tune_step.py --out gpurun_out/r8_tune_ws.jsonl --sm 65536,131072,262144,524288:32,64,128:64,128 --pull "" > gpurun_out/r8_tune_ws.log 2>&1
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29582 tools/timeline.py --engine sm --chunk 262144 --cta 64 --out gpurun_out/r8_tl > gpurun_out/r8_timeline.log 2>&1
true
