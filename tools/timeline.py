"""Per-transfer %globaltimer timeline of one 1F1B step (cfg.trace bit 0), one process per
GPU.  Writes gpurun_out/timeline.r<rank>.json; --show prints a merged table.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/timeline.py [--engine sm|pull]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--engine", default="sm")
ap.add_argument("--chunk", type=int, default=1 << 20)
ap.add_argument("--cta", type=int, default=0)
ap.add_argument("--M", type=int, default=8)
ap.add_argument("--out", default="gpurun_out/timeline")
ap.add_argument("--zc", type=int, default=0)
ap.add_argument("--graph", type=int, default=0, help="time a CUDA-graph replay of the step")
a = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
n = 4096 * 4096 * 2
M = a.M
eng = {"sm": ppc.ENGINE_SM, "ce": ppc.ENGINE_CE, "pull": ppc.ENGINE_PULL}[a.engine]
cfg = ppc.make_config(pp=world, max_msg_bytes=n, chunk_bytes=a.chunk, engine=eng,
                      cta_per_channel=a.cta, trace=1)
comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
X = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)] if rank == 0 else None
G = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)] if rank == world - 1 else None
OUT = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
sa = ppc.StepArgs(M, n, n, x=X, g=G, y=OUT if rank == world - 1 else None,
                  dx=OUT if rank == 0 else None)
s = torch.cuda.current_stream()
if a.zc:
    ppc.register_tensors(comm, X or G)
for _ in range(3):
    ppc.step_1f1b(comm, sa, s)
torch.cuda.synchronize()
dist.barrier()
n_before = len(comm.trace())
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
if a.graph:   # records captured once; each replay rewrites them
    sg = ppc.StepGraph([comm], [sa], [s])
    for _ in range(3):
        sg.launch()
    torch.cuda.synchronize()
    dist.barrier()
    ev0.record(s)
    sg.launch()
    ev1.record(s)
else:
    ev0.record(s)
    ppc.step_1f1b(comm, sa, s)
    ev1.record(s)
torch.cuda.synchronize()
recs = comm.trace()[n_before:]
out = {"rank": rank, "step_ms": ev0.elapsed_time(ev1), "records": recs}
os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
with open(f"{a.out}.r{rank}.json", "w") as fh:
    json.dump(out, fh)
dist.barrier()
if rank == 0:
    allr = []
    for r in range(world):
        d = json.load(open(f"{a.out}.r{r}.json"))
        for x in d["records"]:
            x["rank"] = r
            allr.append(x)
    # %globaltimer is per GPU (offsets between GPUs are arbitrary): times are rank-relative
    t0s = {r: min(x["t_start_ns"] for x in allr if x["rank"] == r) for r in range(world)}
    allr.sort(key=lambda x: (x["rank"], x["t_start_ns"]))
    print(f"step_ms rank0 {out['step_ms']:.3f}")
    for x in allr:
        t0 = t0s[x["rank"]]
        print(f"r{x['rank']} {'send' if x['kind'] == 0 else 'recv'} {x['src']}->{x['dst']} seq {x['seq']} "
              f"mb {x['mb']} start {(x['t_start_ns'] - t0) / 1e3:8.1f} us end "
              f"{(x['t_end_ns'] - t0) / 1e3:8.1f} us dur {(x['t_end_ns'] - x['t_start_ns']) / 1e3:6.1f}")
comm.disconnect()
dist.barrier()
comm.destroy()
dist.destroy_process_group()
