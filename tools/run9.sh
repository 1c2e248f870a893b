timeout 900 python -m pytest tests/test_gpu_local.py tests/test_gpu_toy.py -x -q > gpurun_out/r9_tests.log 2>&1; echo rc=$? >> gpurun_out/r9_tests.log
timeout 200 python bench.py > gpurun_out/r9_bench1.log 2>&1
PPC_LOCAL_DIRECT=0 timeout 200 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r9_bench1_ring.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus 2 --chunk 524288 --cta 64 > gpurun_out/r9_bench2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 bench_exposure.py --layers 1 --out gpurun_out/r9_exposure.jsonl > gpurun_out/r9_exposure.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29593 bench_exposure.py --layers 4 --out gpurun_out/r9_exposure.jsonl >> gpurun_out/r9_exposure.log 2>&1
timeout 120 python tools/xdev_push.py --size 32M --n 4 --cta 64 --chunk 512K > gpurun_out/r9_plain_xdev.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:push -s 6 -c 2 -o gpurun_out/r9_prof_xdev_ws python tools/xdev_push.py --size 32M --n 4 --cta 64 --chunk 512K > gpurun_out/r9_ncu_xdev.log 2>&1
timeout 120 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r9_plain_b1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:copy_kernel -s 20 -c 2 -o gpurun_out/r9_prof_n1_copy python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r9_ncu_n1.log 2>&1
timeout 120 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r9_plain_b2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9_launches_n1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r9_ncu_launch.log 2>&1
true
