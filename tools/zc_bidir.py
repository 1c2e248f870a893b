"""Bidirectional zero-copy message stream probe (torchrun, 2 ranks):
    tools/zc_bidir.py CTAS N [CHUNK_KIB]
Every receive of a direction is enqueued before its sends (bench_sweep's bidir mode)."""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
ctas, N = int(sys.argv[1]), int(sys.argv[2])
chunk = (int(sys.argv[3]) if len(sys.argv) > 3 else 256) << 10
os.environ["PPC_RECV_CTAS"] = str(ctas)
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
n = 32 << 20
cfg = ppc.make_config(pp=world, max_msg_bytes=n, chunk_bytes=chunk, timeout_ns=3_000_000_000)
comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
src = torch.empty(n, dtype=torch.uint8, device="cuda")
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
ppc.register_tensors(comm, [src])
s_send, s_recv = torch.cuda.Stream(), torch.cuda.Stream()
d_out = ppc.FWD if rank == 0 else ppc.BWD
d_in = ppc.BWD if rank == 0 else ppc.FWD
torch.cuda.synchronize()
dist.barrier()
t0 = time.time()
for i in range(N):
    comm.recv(d_in, dst, n, mb=i, stream=s_recv)
for i in range(N):
    comm.send(d_out, src, n, mb=i, stream=s_send)
torch.cuda.synchronize()
print(f"rank {rank} ctas {ctas} N {N} chunk {chunk >> 10}K pdl {os.environ.get('PPC_PDL', '1')} "
      f"err {comm.error_info()} {time.time() - t0:.2f}s", flush=True)
dist.barrier()
comm.disconnect()
dist.barrier()
comm.destroy()
