"""C5 sweep (BASELINE.json configs[4]): PP send/recv message sweep 64 KiB - 1 GiB,
device-direct (SM engine x CTAs x chunk, CE engine x channels) vs the library ceilings
(cudaMemcpyPeer-style CE copy, NCCL send/recv) and the CPU-forwarding baseline B0
(Megatron-Gloo style: .cpu() -> gloo send/recv -> .cuda()).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 bench_sweep.py --out gpurun_out/sweep.jsonl

Unidirectional: rank 0 sends N back-to-back messages FWD, rank 1 receives; time on the
sender from the first enqueue to ppc_pp_wait_consumed (all data in rank 1's user buffer).
Bidirectional: rank 0 -> 1 FWD and 1 -> 0 BWD at the same time (the 1F1B steady state);
each sender reports its own direction.  GB = 1e9 B.
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

KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/sweep.jsonl")
    ap.add_argument("--sizes", default="64K,256K,1M,4M,16M,28M,32M,64M,128M,256M,512M,1G")
    ap.add_argument("--sm", default="16:1M,32:1M,64:1M,32:256K,64:256K,128:256K,32:4M")
    ap.add_argument("--ce", default="1,2,4,8")
    ap.add_argument("--pull", default="", help="PULL engine specs cta:chunk, e.g. 32:1M,64:1M")
    ap.add_argument("--zc", default="", help="zero-copy specs recv_ctas:chunk[:flags], e.g. "
                                             "64:256K:ab (a = cfg.zc_async, sends complete at "
                                             "publication; b = batched receives, 16 per grid)")
    ap.add_argument("--modes", default="uni,bidir")
    ap.add_argument("--channels", default="1",
                    help="MPDT channel counts C (comma list) applied to every SM / zero-copy spec: "
                         "the message's chunks split into C contiguous ranges, one CTA group each")
    ap.add_argument("--comparators", default="nccl,ce_copy,gloo")
    ap.add_argument("--reps", type=int, default=5)
    return ap.parse_args()


def size_of(s):
    u = {"K": KiB, "M": MiB, "G": GiB}
    return int(s[:-1]) * u[s[-1]] if s[-1] in u else int(s)


def nmsgs(n):
    return 200 if n <= MiB else (40 if n <= 64 * MiB else 10)


def emit(fh, rec):
    fh.write(json.dumps(rec) + "\n")
    fh.flush()


def bench_ppc(comm, rank, sizes, modes, label, reps, fh, zc=False, batch=0):
    s_send = torch.cuda.Stream()
    s_recv = torch.cuda.Stream()
    maxn = max(sizes)
    src = torch.empty(maxn, dtype=torch.uint8, device="cuda")
    dst = torch.empty(maxn, dtype=torch.uint8, device="cuda")
    ppc.fill_payload(src, maxn, 42, 0, 0, rank, 0)
    if zc:                       # registered source: receivers pull it over NVLink
        ppc.register_tensors(comm, [src])
    for mode in modes:
        for n in sizes:
            N = nmsgs(n)
            best, times = None, []
            for rep in range(reps + 1):
                sender = rank == 0 or mode == "bidir"
                receiver = rank == 1 or mode == "bidir"
                d_out = ppc.FWD if rank == 0 else ppc.BWD
                d_in = ppc.BWD if rank == 0 else ppc.FWD
                torch.cuda.synchronize()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                if receiver and batch:       # ppc_pp_recv_batch: `batch` messages per grid
                    k0 = min(batch, N)           # distinct destinations inside one grid
                    dsts = [dst] + [torch.empty(n, dtype=torch.uint8, device="cuda")
                                    for _ in range(k0 - 1)]
                    for i0 in range(0, N, batch):
                        k = min(batch, N - i0)
                        comm.recv_batch(d_in, dsts[:k], n, mb0=i0, stream=s_recv)
                elif receiver:
                    for i in range(N):
                        comm.recv(d_in, dst, n, mb=i, stream=s_recv)
                if sender:
                    e0.record(s_send)
                    for i in range(N):
                        comm.send(d_out, src, n, mb=i, stream=s_send)
                    comm.wait_consumed(d_out, s_send)
                    e1.record(s_send)
                torch.cuda.synchronize()
                if comm.poll():
                    raise RuntimeError(f"{label} {mode} {n}: {ppc.STATUS[comm.poll()]}")
                if sender and rep > 0:                       # rep 0 = warm-up
                    times.append(e0.elapsed_time(e1) * 1e-3)
            if times:
                t = sorted(times)[len(times) // 2]
                emit(fh, {"impl": label, "mode": mode, "rank": rank, "bytes": n, "msgs": N,
                          "gbps_median": N * n / t / 1e9, "gbps_best": N * n / min(times) / 1e9,
                          "us_per_msg": t / N * 1e6})


def bench_nccl(rank, sizes, reps, fh, pg):
    s = torch.cuda.current_stream()
    for n in sizes:
        N = nmsgs(n)
        t = torch.empty(n, dtype=torch.uint8, device="cuda")
        times = []
        for rep in range(reps + 1):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(N):
                if rank == 0:
                    dist.send(t, 1, group=pg)
                else:
                    dist.recv(t, 0, group=pg)
            e1.record(s)
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1) * 1e-3)
        if rank == 1:
            tm = sorted(times)[len(times) // 2]
            emit(fh, {"impl": "nccl_send_recv", "mode": "uni", "rank": rank, "bytes": n,
                      "msgs": N, "gbps_median": N * n / tm / 1e9,
                      "gbps_best": N * n / min(times) / 1e9, "us_per_msg": tm / N * 1e6})


def bench_ce_copy(rank, sizes, reps, fh):
    """cudaMemcpyPeer-style copy engine ceiling: one process, cuda:0 -> cuda:1."""
    if rank != 0 or torch.cuda.device_count() < 2:
        return
    for n in sizes:
        N = nmsgs(n)
        a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
        b = torch.empty(n, dtype=torch.uint8, device="cuda:1")
        times = []
        for rep in range(reps + 1):
            torch.cuda.synchronize(0)
            torch.cuda.synchronize(1)
            t0 = time.perf_counter()
            for _ in range(N):
                b.copy_(a, non_blocking=True)
            torch.cuda.synchronize(0)
            torch.cuda.synchronize(1)
            if rep:
                times.append(time.perf_counter() - t0)
        tm = sorted(times)[len(times) // 2]
        emit(fh, {"impl": "ce_peer_copy", "mode": "uni", "rank": 0, "bytes": n, "msgs": N,
                  "gbps_median": N * n / tm / 1e9, "gbps_best": N * n / min(times) / 1e9,
                  "us_per_msg": tm / N * 1e6, "timing": "host perf_counter"})


def bench_gloo(rank, sizes, fh):
    """B0: the paper's Megatron-Gloo CPU-forwarding path: D2H, gloo TCP, H2D."""
    for n in [x for x in sizes if x <= 256 * MiB]:
        g = torch.empty(n, dtype=torch.uint8, device="cuda")
        times = []
        for rep in range(3):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            if rank == 0:
                dist.send(g.cpu(), 1)
            else:
                h = torch.empty(n, dtype=torch.uint8)
                dist.recv(h, 0)
                g.copy_(h)
                torch.cuda.synchronize()
            if rep:
                times.append(time.perf_counter() - t0)
        if rank == 1:
            tm = min(times)
            emit(fh, {"impl": "B0_gloo_cpu_forward", "mode": "uni", "rank": 1, "bytes": n,
                      "msgs": 1, "gbps_median": n / tm / 1e9, "gbps_best": n / tm / 1e9,
                      "us_per_msg": tm * 1e6})


def main():
    a = parse()
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    sizes = [size_of(s) for s in a.sizes.split(",")]
    modes = a.modes.split(",")
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    fh = open(a.out.replace(".jsonl", f".r{rank}.jsonl"), "w")
    maxn = max(sizes)
    chans = [int(x) for x in a.channels.split(",")]
    for spec, C in [(x, c) for x in a.sm.split(",") if x and x != "none" for c in chans]:
        cta, chunk = spec.split(":")
        cfg = ppc.make_config(pp=world, max_msg_bytes=maxn, chunk_bytes=size_of(chunk),
                              cta_per_channel=max(1, int(cta) // C), channels=C,
                              engine=ppc.ENGINE_SM)
        comm = ppc.connect_distributed(cfg, rank, world, torch.cuda.current_device(),
                                       with_nccl=False)
        bench_ppc(comm, rank, sizes, modes, f"ppc_sm_cta{cta}_chunk{chunk}_C{C}", a.reps, fh)
        dist.barrier()
        comm.disconnect()
        dist.barrier()
        comm.destroy()
    for ch in [x for x in a.ce.split(",") if x and x != "none"]:
        cfg = ppc.make_config(pp=world, max_msg_bytes=maxn, chunk_bytes=MiB, channels=int(ch),
                              engine=ppc.ENGINE_CE)
        comm = ppc.connect_distributed(cfg, rank, world, torch.cuda.current_device(),
                                       with_nccl=False)
        bench_ppc(comm, rank, sizes, modes, f"ppc_ce_ch{ch}", a.reps, fh)
        dist.barrier()
        comm.disconnect()
        dist.barrier()
        comm.destroy()
    for spec, C in [(x, c) for x in a.zc.split(",") if x for c in chans]:
        parts = spec.split(":")            # recv_ctas:chunk[:flags]  (a = zc_async, b = batch)
        rc, chunk = parts[0], parts[1]
        zc_async = len(parts) > 2 and "a" in parts[2]
        batch = 16 if len(parts) > 2 and "b" in parts[2] else 0
        os.environ["PPC_RECV_CTAS"] = rc
        cfg = ppc.make_config(pp=world, max_msg_bytes=maxn, chunk_bytes=size_of(chunk),
                              zc_async=int(zc_async), channels=C)
        comm = ppc.connect_distributed(cfg, rank, world, torch.cuda.current_device(),
                                       with_nccl=False)
        label = (f"ppc_zerocopy{'_async' if zc_async else ''}{'_batch' if batch else ''}"
                 f"_recv{rc}_chunk{chunk}_C{C}")
        bench_ppc(comm, rank, sizes, modes, label, a.reps, fh, zc=True, batch=batch)
        os.environ.pop("PPC_RECV_CTAS")
        dist.barrier()
        comm.disconnect()
        dist.barrier()
        comm.destroy()
    for spec in [x for x in a.pull.split(",") if x]:
        cta, chunk = spec.split(":")
        cfg = ppc.make_config(pp=world, max_msg_bytes=maxn, chunk_bytes=size_of(chunk),
                              cta_per_channel=int(cta), engine=ppc.ENGINE_PULL)
        comm = ppc.connect_distributed(cfg, rank, world, torch.cuda.current_device(),
                                       with_nccl=False)
        bench_ppc(comm, rank, sizes, modes, f"ppc_pull_cta{cta}_chunk{chunk}", a.reps, fh)
        dist.barrier()
        comm.disconnect()
        dist.barrier()
        comm.destroy()
    comps = a.comparators.split(",")
    if "nccl" in comps:
        pg = dist.new_group(backend="nccl")
        bench_nccl(rank, sizes, a.reps, fh, pg)
    dist.barrier()
    if "ce_copy" in comps:
        bench_ce_copy(rank, sizes, a.reps, fh)
    dist.barrier()
    if "gloo" in comps:
        bench_gloo(rank, sizes, fh)
    dist.barrier()
    fh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
