"""Stability run (§3.3 P:L173 "throughput remains stable
throughout the 500 iterations"): N consecutive comm-only 1F1B steps of the C2 workload, each
timed with CUDA events, reported as a per-step time distribution.

    python bench_stability.py --steps 500                      # virtual stages on one GPU
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 bench_stability.py --steps 500
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_2602_18007_b200 as ppc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--cta", type=int, default=64)
    ap.add_argument("--out", default="gpurun_out/stability.json")
    ap.add_argument("--graph", type=int, default=1, help="replay the step as a CUDA graph")
    ap.add_argument("--zc", type=int, default=1, help="N>=2: zero-copy registered sources")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist_mode = world > 1
    torch.cuda.set_device(rank if dist_mode else 0)
    if dist_mode:
        dist.init_process_group("gloo")
    n, M = 4096 * 4096 * 2, a.M
    # bench.py's launch configuration: zero-copy pulls (256 KiB grain) + CUDA graph at N >= 2
    chunk = a.chunk or (((256 if a.zc else 512) << 10) if dist_mode else (128 << 10))
    cfg = ppc.make_config(pp=2, dp=max(1, world // 2), max_msg_bytes=n, chunk_bytes=chunk,
                          cta_per_channel=a.cta if (dist_mode and not a.zc) else 0)
    if dist_mode:
        comms = [ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)]
        stages = [comms[0].group(ppc.GROUP_PP)[0].index(rank)]
    else:
        comms = ppc.virtual_stages(cfg, 0)
        stages = [0, 1]
    bufs = lambda: [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
    src = {s: bufs() for s in stages}            # X on stage 0, G on stage 1
    args = [ppc.StepArgs(M, n, n, x=src[s] if s == 0 else None, g=src[s] if s == 1 else None,
                         y=bufs() if s == 1 else None, dx=bufs() if s == 0 else None) for s in stages]
    streams = [torch.cuda.Stream() for _ in stages]
    if dist_mode and a.zc:
        ppc.register_tensors(comms[0], src[stages[0]])
    graph = [None]

    def step():
        if graph[0] is not None:
            graph[0].launch()
        elif dist_mode:
            ppc.step_1f1b(comms[0], args[0], streams[0])
        else:
            ppc.step_1f1b_local(comms, args, streams)

    step()
    torch.cuda.synchronize()
    if a.graph:
        graph[0] = ppc.StepGraph(comms, args, streams)
        streams = streams[:1]             # a graph replay is timed on its launch stream
        stages = stages[:1]
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    if dist_mode:
        dist.barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)] for _ in stages]
    for k, st in enumerate(streams):
        ev[k][0].record(st)
    for i in range(a.steps):
        step()
        for k, st in enumerate(streams):
            ev[k][i + 1].record(st)
    torch.cuda.synchronize()
    per = [max(ev[k][i].elapsed_time(ev[k][i + 1]) for k in range(len(stages))) for i in range(a.steps)]
    if dist_mode:
        t = torch.tensor(per, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per = t.tolist()
    q = sorted(per)
    pct = lambda p: q[min(len(q) - 1, int(p * len(q)))]
    rec = {"workload": "C2 PP=2 [1,4096,4096] bf16 M=8 comm-only", "n_gpus": world,
           "cuda_graph": bool(a.graph), "zero_copy": bool(dist_mode and a.zc),
           "steps": a.steps, "ms_mean": statistics.mean(per), "ms_p50": pct(0.5),
           "ms_p90": pct(0.9), "ms_p99": pct(0.99), "ms_min": q[0], "ms_max": q[-1],
           "cv": statistics.pstdev(per) / statistics.mean(per),
           "tokens_per_s_mean": (world // 2 or 1) * M * 4096 / (statistics.mean(per) * 1e-3),
           "errors": [c.poll() for c in comms if c.poll()]}
    if rank == 0:
        print(json.dumps(rec), flush=True)
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "w") as fh:
            json.dump({**rec, "per_step_ms": per}, fh)
    if graph[0] is not None:
        graph[0].destroy()
    for c in comms:
        c.disconnect()
    if dist_mode:
        dist.barrier()
    for c in comms:
        c.destroy()
    if dist_mode:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
