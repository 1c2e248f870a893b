python tools/graph_debug.py > gpurun_out/r15_gdbg.log 2>&1
PPC_DEBUG=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 tests/mp_worker.py graph > gpurun_out/r15_mp_graph.log 2>&1; echo rc=$? >> gpurun_out/r15_mp_graph.log
true
