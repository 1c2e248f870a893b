"""Debug harness for ppc_pp_recv_gather (torchrun, 2 or 4 ranks): FWD only, short timeouts."""
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
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
cfg = ppc.make_config(tp=tp, pp=world // tp, dp=1, max_msg_bytes=4 << 20, chunk_bytes=256 << 10,
                      timeout_ns=3_000_000_000)
comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
pp_i, tp_i = rank // tp, rank % tp
slice_n = 256 << 10
total = tp * slice_n
full = torch.empty(total, dtype=torch.uint8, device="cuda")
ppc.fill_payload(full, total, 42, 0, 0xFF, 0, 0)
ppc.register_tensors(comm, [full])
out = torch.zeros(total, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
s2 = torch.cuda.Stream()
if pp_i == 0:
    comm.send(ppc.FWD, full.data_ptr() + tp_i * slice_n, slice_n, mb=0, stream=s2)
else:
    comm.recv_gather(ppc.FWD, out, total, mb=0, stream=s)
torch.cuda.synchronize()
ok = True
if pp_i == 1:
    ok = np.array_equal(out.cpu().numpy(), P.payload_bytes(42, 0, 0xFF, 0, 0, total))
print(f"rank {rank} tp {tp} err {comm.error_info()} data_ok {ok}", flush=True)
dist.barrier()
comm.disconnect()
dist.barrier()
comm.destroy()
