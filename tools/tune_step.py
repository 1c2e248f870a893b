"""Grid/chunk tuning of the C2 1F1B comm-only step on 2 GPUs (one torchrun session, many
configs).  Prints one JSON line per config (rank 0): step time (CUDA events, max over ranks).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/tune_step.py --out gpurun_out/tune.jsonl
"""
import argparse
import itertools
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default="gpurun_out/tune.jsonl")
ap.add_argument("--sm", default="131072,262144,524288,1048576:32,64,128:64,128")
ap.add_argument("--pull", default="131072,262144,1048576:32,64,128:128")
ap.add_argument("--zc", default="262144,524288,1048576:32,64,128")
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
n, M = 4096 * 4096 * 2, 8
X = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)] if rank == 0 else None
G = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)] if rank == 1 else None
OUT = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
sa = ppc.StepArgs(M, n, n, x=X, g=G, y=OUT if rank == 1 else None, dx=OUT if rank == 0 else None)
s = torch.cuda.current_stream()
fh = open(a.out, "w") if rank == 0 else None


def run(engine, chunk, cta, extra_env, zc=False):
    for k, v in extra_env.items():
        os.environ[k] = str(v)
    cfg = ppc.make_config(pp=2, max_msg_bytes=n, chunk_bytes=chunk, engine=engine, cta_per_channel=cta)
    comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
    if zc:
        ppc.register_tensors(comm, X or G)
    extra_env = dict(extra_env, zc=int(zc))
    for _ in range(3):
        ppc.step_1f1b(comm, sa, s)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(a.steps):
        ppc.step_1f1b(comm, sa, s)
    e1.record(s)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / a.steps], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = comm.poll() == 0
    dist.barrier()
    comm.disconnect()
    dist.barrier()
    comm.destroy()
    for k in extra_env:
        os.environ.pop(k, None)
    rec = {"engine": engine, "chunk": chunk, "cta": cta, **extra_env, "us_per_step": t.item() * 1e3,
           "mtok_s": M * 4096 / (t.item() * 1e-3) / 1e6, "ok": ok}
    if fh:
        fh.write(json.dumps(rec) + "\n")
        fh.flush()
        print(json.dumps(rec), flush=True)


def grid(spec):
    if not spec:
        return []
    parts = [[int(x) for x in p.split(",")] for p in spec.split(":")]
    return list(itertools.product(*parts))


for chunk, cta, rc in grid(a.sm):
    run(ppc.ENGINE_SM, chunk, cta, {"PPC_RECV_CTAS": rc})
for chunk, cta, st in grid(a.pull):
    run(ppc.ENGINE_PULL, chunk, cta, {"PPC_STAGE_CTAS": st})
for chunk, rc in grid(a.zc):     # zero-copy pulls: chunk = pull grain, rc = pulling CTAs
    run(ppc.ENGINE_SM, chunk, 0, {"PPC_RECV_CTAS": rc}, zc=True)
dist.destroy_process_group()
