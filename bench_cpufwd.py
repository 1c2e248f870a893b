"""1F1B tokens/s: device-direct (libppc) vs CPU-Forwarding (B1 = libppcb pinned /dev/shm ring
with 1-8 channels, B0 = Megatron-Gloo style .cpu() -> gloo -> .cuda()), plus the B1 per-message
sweep.  BASELINE.json metric "1F1B tokens/s device-direct vs CPU-fwd", configs[1] shape
(PP=2, [1,4096,4096] bf16, M=8).  Two processes, one per GPU:

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 bench_cpufwd.py --out gpurun_out/cpufwd.jsonl
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import paper_2602_18007_b200 as ppc  # noqa: E402
from paper_2602_18007_b200.cpufwd import CpuFwdLink  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/cpufwd.jsonl")
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--seq", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--channels", default="1,2,4,8")
    ap.add_argument("--chunk", type=int, default=4 << 20)
    ap.add_argument("--skip-b0", action="store_true")
    return ap.parse_args()


def main():
    a = parse()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    assert world == 2, "PP=2 pair"
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    n = a.seq * a.hidden * 2
    M = a.M
    ops = ppc.schedule_1f1b(2, rank, M)
    X = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)] if rank == 0 else None
    G = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)] if rank == 1 else None
    OUT = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
    for m in range(M):
        if X:
            ppc.fill_payload(X[m], n, 42, 0, 0xFF, 0, m)
        if G:
            ppc.fill_payload(G[m], n, 42, 0, 0xFF, 1, m)
    torch.cuda.synchronize()
    fh = open(a.out.replace(".jsonl", f".r{rank}.jsonl"), "w") if rank == 0 else None

    def record(rec):
        if fh:
            fh.write(json.dumps(rec) + "\n")
            fh.flush()
            print(json.dumps(rec), flush=True)

    def check():
        ref = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in (0, M - 1)]
        for r, m in zip(ref, (0, M - 1)):
            ppc.fill_payload(r, n, 42, 0, 0xFF, 1 if rank == 0 else 0, m)
        return all(torch.equal(OUT[m], r) for r, m in zip(ref, (0, M - 1)))

    def timed(step_fn, steps):
        step_fn()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            step_fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        t = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item() / steps

    base = {"M": M, "msg_bytes": n, "pp": 2, "workload": "C2 PP=2 [1,4096,4096] bf16 M=8 comm-only"}

    # ---- device-direct (libppc step driver)
    cfg = ppc.make_config(pp=2, max_msg_bytes=n, chunk_bytes=1 << 20)
    comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
    sa = ppc.StepArgs(M, n, n, x=X, g=G, y=OUT if rank == 1 else None, dx=OUT if rank == 0 else None)
    s = torch.cuda.current_stream()
    t = timed(lambda: ppc.step_1f1b(comm, sa, s), 20)
    ok = check()
    record({**base, "impl": "device_direct_ppc", "s_per_step": t, "tokens_per_s": M * a.seq / t,
            "outputs_ok": ok, "timing": "host wall clock, max over ranks"})
    dist.barrier()
    comm.disconnect()
    dist.barrier()
    comm.destroy()

    # ---- B1: pinned shm ring, C channels
    for C in [int(x) for x in a.channels.split(",")]:
        tags = [None, None]
        dist.all_gather_object(tags, os.getpid())      # unique shm names per run
        fwd = CpuFwdLink(f"fwd{C}_{tags[0]}", rank == 0, n, a.chunk, 2, C, rank)
        bwd = CpuFwdLink(f"bwd{C}_{tags[1]}", rank == 1, n, a.chunk, 2, C, rank)
        dist.barrier()
        fwd.connect()
        bwd.connect()
        dist.barrier()

        def b1_step():
            for kind, m in ops:
                if rank == 0:
                    if kind == "F":
                        fwd.send(X[m], n, m, s)
                    else:
                        bwd.recv(OUT[m], n, m, s)
                else:
                    if kind == "F":
                        fwd.recv(OUT[m], n, m, s)
                    else:
                        bwd.send(G[m], n, m, s)

        t = timed(b1_step, a.steps)
        ok = check()
        record({**base, "impl": f"B1_cpu_forward_shm_ch{C}", "channels": C, "chunk": a.chunk,
                "s_per_step": t, "tokens_per_s": M * a.seq / t, "outputs_ok": ok,
                "timing": "host wall clock, max over ranks"})
        # per-message unidirectional sweep (C5 CPU-forwarding leg)
        for sz in (1 << 20, 32 << 20, n):
            N = 10
            dist.barrier()
            t0 = time.perf_counter()
            for i in range(N):
                if rank == 0:
                    fwd.send(X[0], sz, i, s)
                else:
                    fwd.recv(OUT[0], sz, i, s)
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            record({"impl": f"B1_cpu_forward_shm_ch{C}", "mode": "uni", "bytes": sz, "msgs": N,
                    "gbps": N * sz / dt.item() / 1e9})
        dist.barrier()
        fwd.destroy()
        bwd.destroy()
        dist.barrier()

    # ---- B0: Megatron-Gloo style
    if not a.skip_b0:
        peer = 1 - rank

        def b0_step():
            reqs, keep = [], []
            for kind, m in ops:
                if (rank == 0 and kind == "F") or (rank == 1 and kind == "B"):
                    h = (X if rank == 0 else G)[m].cpu()
                    keep.append(h)
                    reqs.append(dist.isend(h, peer))
                else:
                    h = torch.empty(n, dtype=torch.uint8)
                    dist.recv(h, peer)
                    OUT[m].copy_(h)
            for r in reqs:
                r.wait()

        t = timed(b0_step, 2)
        ok = check()
        record({**base, "impl": "B0_gloo_cpu_forward", "s_per_step": t,
                "tokens_per_s": M * a.seq / t, "outputs_ok": ok,
                "timing": "host wall clock, max over ranks"})
    if fh:
        fh.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
