set -x
timeout 300 python -m pytest tests/test_gpu_local.py -x -q > gpurun_out/r3_gpu_local.log 2>&1; echo rc=$? >> gpurun_out/r3_gpu_local.log
for sz in 32M 1G; do for cta in 16 32 64; do for mode in uni bidir; do
  timeout 60 python tools/xdev_push.py --size $sz --n 20 --cta $cta --chunk 1M --mode $mode >> gpurun_out/r3_xdev.jsonl 2>>gpurun_out/r3_xdev.err
done; done; done
timeout 60 python tools/xdev_push.py --size 32M --n 20 --engine ce --channels 2 >> gpurun_out/r3_xdev.jsonl 2>>gpurun_out/r3_xdev.err
timeout 120 python bench.py --no-cpu-baseline > gpurun_out/r3_bench1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --no-e2e > gpurun_out/r3_bench2.log 2>&1
timeout 120 python tools/xdev_push.py --size 32M --n 4 --cta 32 > gpurun_out/r3_plain_xdev.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:push_kernel -s 6 -c 2 -o gpurun_out/prof_xdev_push python tools/xdev_push.py --size 32M --n 4 --cta 32 > gpurun_out/r3_ncu_xdev.log 2>&1
timeout 120 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_plain_b1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"push_kernel|recv_kernel" -s 40 -c 4 -o gpurun_out/prof_n1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_ncu_n1.log 2>&1
timeout 120 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_plain_b2.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r3_ncu_launch.log 2>&1
true
