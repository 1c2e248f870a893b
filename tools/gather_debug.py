"""Debug harness for ppc_pp_recv_gather (torchrun): tools/gather_debug.py TP BOTH M"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402
from synth import payload as P  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
tp = int(sys.argv[1]) if len(sys.argv) > 1 else 2
both = int(sys.argv[2]) if len(sys.argv) > 2 else 0
M = int(sys.argv[3]) if len(sys.argv) > 3 else 1
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
cfg = ppc.make_config(tp=tp, pp=world // tp, dp=1, max_msg_bytes=4 << 20, chunk_bytes=256 << 10,
                      timeout_ns=3_000_000_000)
comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
pp_i, tp_i = rank // tp, rank % tp
slice_n = 256 << 10
total = tp * slice_n
d_send = ppc.FWD if pp_i == 0 else ppc.BWD
d_recv = 1 - d_send
fulls = [torch.empty(total, dtype=torch.uint8, device="cuda") for _ in range(M)]
for m in range(M):
    ppc.fill_payload(fulls[m], total, 42, 0, 0xFF, d_send, m)
ppc.register_tensors(comm, fulls)
outs = [torch.zeros(total, dtype=torch.uint8, device="cuda") for _ in range(M)]
s = torch.cuda.Stream()
s2 = torch.cuda.Stream()
for m in range(M):
    if pp_i == 0 or both:
        comm.send(d_send, fulls[m].data_ptr() + tp_i * slice_n, slice_n, mb=m, stream=s2)
    if pp_i == 1 or both:
        comm.recv_gather(d_recv, outs[m], total, mb=m, stream=s)
torch.cuda.synchronize()
ok = True
if pp_i == 1 or both:
    ok = all(np.array_equal(outs[m].cpu().numpy(), P.payload_bytes(42, 0, 0xFF, d_recv, m, total))
             for m in range(M))
print(f"rank {rank} tp {tp} both {both} M {M} err {comm.error_info()} data_ok {ok}", flush=True)
dist.barrier()
comm.disconnect()
dist.barrier()
comm.destroy()
