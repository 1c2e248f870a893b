set -x
./tools/nvlink_probe > gpurun_out/r4_probe.jsonl 2> gpurun_out/r4_probe.err
timeout 600 python -m pytest tests/test_gpu_toy.py -x -q > gpurun_out/r4_toy.log 2>&1; echo rc=$? >> gpurun_out/r4_toy.log
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "toy" > gpurun_out/r4_toy_mp.log 2>&1; echo rc=$? >> gpurun_out/r4_toy_mp.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench_cpufwd.py --out gpurun_out/r4_cpufwd.jsonl > gpurun_out/r4_cpufwd.log 2>&1; echo rc=$? >> gpurun_out/r4_cpufwd.log
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/r4_lscpu.txt
true
