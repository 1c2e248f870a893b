"""Where the N=2 C2 step's per-hop time goes: per-CTA %globaltimer stamps of every zero-copy
receive kernel (PPC_DBG_STAMPS=1, eager steps), two ranks (torchrun, one GPU each).

    PPC_DBG_STAMPS=1 torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/hop_stamps.py

Per receive kernel (rank, seq): the spread of its CTAs' release from griddepcontrol.wait,
header-seen, first-chunk and done times, and the gap from the previous receive kernel's
last CTA on the same GPU (the kernel boundary).  Cross-GPU gaps (the peer's publication ->
our header seen) assume the GPUs' %globaltimer agree, which is only approximately true.
Prints one JSON summary line (rank 0) and writes gpurun_out/hop_stamps.json."""
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402


def main():
    assert os.environ.get("PPC_DBG_STAMPS") == "1", "run with PPC_DBG_STAMPS=1"
    graph = "--graph" in sys.argv          # time CUDA-graph replays (the bench's mode)
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    n, M = 4096 * 4096 * 2, 8
    cfg = ppc.make_config(pp=2, max_msg_bytes=n, chunk_bytes=256 << 10)
    comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
    X = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)] if rank == 0 else None
    G = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)] if rank == 1 else None
    for m in range(M):
        if X:
            ppc.fill_payload(X[m], n, 42, 0, 0xFF, 0, m)
        if G:
            ppc.fill_payload(G[m], n, 42, 0, 0xFF, 1, m)
    torch.cuda.synchronize()
    ppc.register_tensors(comm, X or G)
    out = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
    args = ppc.StepArgs(M, n, n, x=X, g=G, y=out if rank == 1 else None, dx=out if rank == 0 else None)
    s = torch.cuda.Stream()
    times = []
    g = None
    if graph:                              # eager step first (buffers), then the capture
        ppc.step_1f1b(comm, args, s)
        torch.cuda.synchronize()
        dist.barrier()
        g = ppc.StepGraph([comm], [args], [s])
    for step in range(6):
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        if g:
            g.launch()
        else:
            ppc.step_1f1b(comm, args, s)
        e1.record(s)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) * 1e3)
    if g:
        g.destroy()
    st = comm.debug_stamps()
    allst = [None] * world
    dist.all_gather_object(allst, st)
    if rank == 0:
        launches = []
        for r, lst in enumerate(allst):
            for seq, d, g, rows in lst:
                rows = [x for x in rows if all(x)]
                if not rows:
                    continue
                for x in rows:                     # [2]: SM id << 48 | timer low 48 bits
                    x.append(x[2] >> 48)
                    x[2] = (x[1] & ~0xFFFFFFFFFFFF) | (x[2] & 0xFFFFFFFFFFFF)
                col = lambda k: [x[k] for x in rows]
                launches.append({"rank": r, "seq": seq, "dir": d, "ctas": len(rows),
                                 "cta_sm_done": [(x[4], x[3] - min(col(1))) for x in rows],
                                 "rel_min": min(col(0)), "rel_max": max(col(0)),
                                 "seen_min": min(col(1)), "seen_max": max(col(1)),
                                 "first_min": min(col(2)) if all(col(2)) else None,
                                 "done_min": min(col(3)), "done_max": max(col(3))})
        per = {}
        for L in launches:
            per.setdefault(L["rank"], []).append(L)
        hops = []
        for r, lst in per.items():
            lst.sort(key=lambda L: L["rel_min"])
            # eager: the last steps; graph: the captured launches (the last replay's stamps)
            last_steps = lst[-M:] if graph else [L for L in lst if L["seq"] > 2 * M]
            for prev, cur in zip(last_steps, last_steps[1:]):
                hops.append({"rank": r, "seq": cur["seq"],
                             "boundary_us": (cur["rel_min"] - prev["done_max"]) * 1e-3,
                             "release_spread_us": (cur["rel_max"] - cur["rel_min"]) * 1e-3,
                             "rel_to_seen_us": (cur["seen_min"] - cur["rel_min"]) * 1e-3,
                             "seen_spread_us": (cur["seen_max"] - cur["seen_min"]) * 1e-3,
                             "pull_us": (cur["done_max"] - cur["seen_min"]) * 1e-3,
                             "tail_us": (cur["done_max"] - cur["done_min"]) * 1e-3})
        med = lambda k: statistics.median(h[k] for h in hops)
        # per SM: mean (done - first header seen) over the analysed launches
        by_sm = {}
        for r, lst in per.items():
            for L in (lst[-M:] if graph else [L for L in lst if L["seq"] > 2 * M]):
                for sm, t in L["cta_sm_done"]:
                    by_sm.setdefault(sm, []).append(t * 1e-3)
        sm_mean = sorted((statistics.mean(v), sm) for sm, v in by_sm.items())
        summary = {"graph": graph, "step_us": times[2:], "hops": len(hops),
                   "sm_done_us": {"fastest": sm_mean[:5], "slowest": sm_mean[-5:],
                                  "n_sms": len(sm_mean)},
                   "median": {k: med(k) for k in ("boundary_us", "release_spread_us",
                                                  "rel_to_seen_us", "seen_spread_us",
                                                  "pull_us", "tail_us")}}
        print(json.dumps(summary), flush=True)
        os.makedirs("gpurun_out", exist_ok=True)
        with open("gpurun_out/hop_stamps.json", "w") as fh:
            json.dump({"summary": summary, "hops": hops, "launches": launches}, fh)
    dist.barrier()
    comm.disconnect()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
