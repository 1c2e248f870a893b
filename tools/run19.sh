timeout 300 python bench.py > gpurun_out/r19_bench1.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 2 > gpurun_out/r19_bench2.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 bench.py --gpus 4 > gpurun_out/r19_bench4.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29693 bench.py --gpus 4 --pp 4 --M 16 --no-e2e > gpurun_out/r19_bench4_pp4_m16.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29694 bench.py --gpus 4 --pp 4 --M 32 --hidden 3584 --no-e2e > gpurun_out/r19_bench4_pp4_m32_qwen.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r19_reference.log 2>&1
timeout 120 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r19_plain_b.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r19_launches_n1.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r19_ncu_launch.log 2>&1
timeout 120 python tools/xdev_push.py --size 32M --n 4 --engine pull --cta 64 --chunk 256K > gpurun_out/r19_plain_xdev.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:recv_kernel -s 6 -c 2 -o gpurun_out/r19_prof_pull python tools/xdev_push.py --size 32M --n 4 --engine pull --cta 64 --chunk 256K > gpurun_out/r19_ncu_pull.log 2>&1
true
