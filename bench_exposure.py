"""Exposed PP communication in a compute-bearing 1F1B step (BASELINE.json target "exposed PP
communication < 5% of 1F1B step time"; R13 / R19), optionally with DCBS tensor
parallelism under load (TP traffic on NCCL inside the stage
compute, PP traffic on libppc's kernels, both on the same NVLink egress).

Stage compute = L LLaMA-8B-shaped MLP blocks per stage on the boundary tensor [4096, 4096]
bf16 (h = 4096, ffn = 14336): x @ W1 -> silu -> @ W2; backward runs the same GEMMs twice.
With --tp T the block is Megatron-split: W1 column-split [h, ffn/T], W2 row-split
[ffn/T, h], and every pass of a block ends with TWO in-place NCCL allreduces of the
[4096, 4096] bf16 partial sums over the TP group through ppc_allreduce (the MLP's and a
stand-in for attention's) — issued on the stage stream by the stage fn, so
they run beside libppc's PP kernels.  cuBLAS via torch is the *user's model*; the transfers
are libppc's.  exposed = (T_step - T_step,flags-only) / T_step, where the control run uses
the same schedule, streams, flags and NCCL traffic with zero-byte PP messages.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 bench_exposure.py --pp 2 --tp 2 --M 16
    torchrun --nproc-per-node 4 ... bench_exposure.py --pp 4 --M 16 --layers 8
    torchrun --nproc-per-node 2 ... bench_exposure.py --layer-times     # per-layer fwd / bwd ms

--layer-times also times one block's forward and backward alone (CUDA events, median of 10)
on every rank, the measured per-layer costs the partition planner consumes (NEXT-3).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import paper_2602_18007_b200 as ppc  # noqa: E402

NCCL_BF16 = 9


class _CAI:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<u2", "data": (ptr, False),
                                         "version": 3, "strides": None}


def as_bf16(ptr, numel):
    return torch.as_tensor(_CAI(ptr, numel), device="cuda").view(torch.bfloat16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pp", type=int, default=0, help="0 = world / tp")
    ap.add_argument("--tp", type=int, default=1)
    ap.add_argument("--layers", type=int, default=1, help="MLP blocks per stage")
    ap.add_argument("--layers-per-stage", default="",
                    help="comma list, one count per stage (overrides --layers): uneven splits")
    ap.add_argument("--ffn-scale-stage0", type=float, default=1.0,
                    help="stage 0's ffn width x this (a slower stage, the paper's AMD side)")
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--ffn", type=int, default=14336)
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--reps", type=int, default=3, help="alternating full / control repeats")
    ap.add_argument("--engine", default="sm")
    ap.add_argument("--layer-times", action="store_true")
    ap.add_argument("--comm-gbps", type=float, default=643.0,
                    help="planner: per-message transfer rate (measured N=2 pull data phase)")
    ap.add_argument("--out", default="gpurun_out/exposure.jsonl")
    ap.add_argument("--inplace", action="store_true",
                    help="PPC_STEP_INPLACE=1: stage fns produce straight into the peer's slot")
    a = ap.parse_args()
    if a.inplace:
        os.environ["PPC_STEP_INPLACE"] = "1"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    TP = a.tp
    S = a.pp or world // TP
    assert world % (S * TP) == 0
    M, T, H, F = a.M, 4096, a.hidden, a.ffn // TP
    nbytes = T * H * 2
    per_stage = [int(x) for x in a.layers_per_stage.split(",")] if a.layers_per_stage else [a.layers] * S
    assert len(per_stage) == S
    stage_of = lambda r: r // (TP * (world // (S * TP)))      # rank = pp_i * tp * dp + ...
    L = per_stage[stage_of(rank)]
    if stage_of(rank) == 0:
        F = int(round(F * a.ffn_scale_stage0 / 64)) * 64
    g = torch.Generator(device="cuda").manual_seed(42 + rank)
    W1 = [torch.randn(H, F, device="cuda", dtype=torch.bfloat16, generator=g) * 0.02
          for _ in range(L)]
    W2 = [torch.randn(F, H, device="cuda", dtype=torch.bfloat16, generator=g) * 0.02
          for _ in range(L)]
    x0 = torch.randn(T, H, device="cuda", dtype=torch.bfloat16, generator=g)
    eng = {"sm": ppc.ENGINE_SM, "pull": ppc.ENGINE_PULL, "ce": ppc.ENGINE_CE}[a.engine]
    cfg = ppc.make_config(tp=TP, pp=S, dp=world // (S * TP), max_msg_bytes=nbytes,
                          chunk_bytes=1 << 20, engine=eng)
    comm = ppc.connect_distributed(cfg, rank, world, local, with_nccl=TP > 1)
    stage = comm.group(ppc.GROUP_PP)[0].index(rank)
    n_ar = [0]

    def block(h, l, out):
        y = torch.matmul(torch.nn.functional.silu(h @ W1[l]), W2[l], out=out)
        if TP > 1:      # DCBS: TP partial sums on NCCL, on the stage stream
            s = torch.cuda.current_stream().cuda_stream
            comm.allreduce(ppc.GROUP_TP, y, NCCL_BF16, stream=s)
            comm.allreduce(ppc.GROUP_TP, y, NCCL_BF16, stream=s)
            n_ar[0] += 2
        return y

    def compute(inp, out, reps, stream):
        with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
            h = x0 if inp is None else inp.view(T, H)
            for r in range(reps):
                for l in range(L):
                    last = out is not None and r == reps - 1 and l == L - 1
                    # the last GEMM's epilogue stores straight into `out` (with
                    # PPC_STEP_INPLACE: the receiver's ring slot, over NVLink)
                    h = block(h, l, out.view(T, H) if last else None)

    def fwd(user, mb, inp, out, ib, ob, stream):
        compute(as_bf16(inp, T * H) if inp and ib else None,
                as_bf16(out, T * H) if out and ob else None, 1, stream)
        return 0

    def bwd(user, mb, inp, out, ib, ob, stream):
        compute(as_bf16(inp, T * H) if inp and ib else None,
                as_bf16(out, T * H) if out and ob else None, 2, stream)
        return 0

    s = torch.cuda.Stream()
    layer = None
    if a.layer_times:
        # sustained per-layer time: the mean over ~1 s of back-to-back blocks (a power-capped
        # B200 runs a long GEMM stream — the pipeline step — below its burst clock, and a
        # short timed burst after idle over-states the rate); bwd = 2 blocks (the proxy's bwd)
        ts = {"fwd": [], "bwd": []}
        with torch.cuda.stream(s):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            block(x0, 0, None)
            e1.record(s)
            torch.cuda.synchronize()
            n_blk = torch.tensor([max(10, int(1000.0 / max(e0.elapsed_time(e1), 0.05)))])
            dist.all_reduce(n_blk, op=dist.ReduceOp.MAX)     # TP ranks call NCCL in lockstep
            n_blk = int(n_blk.item())
            for _ in range(3):
                e0.record(s)
                for _ in range(n_blk):
                    block(x0, 0, None)
                e1.record(s)
                torch.cuda.synchronize()
                ts["fwd"].append(e0.elapsed_time(e1) / n_blk)
                ts["bwd"].append(2 * e0.elapsed_time(e1) / n_blk)
        layer = {k: statistics.median(v) for k, v in ts.items()}

    res = {"full": [], "flags_only": []}
    args = {label: ppc.StepArgs(M, msg, msg, fwd=fwd, bwd=bwd)
            for label, msg in (("full", nbytes), ("flags_only", 0))}
    for label in ("full", "flags_only"):        # warm both (allocations, cuBLAS handles)
        ppc.step_1f1b(comm, args[label], s)
    torch.cuda.synchronize()
    n_ar[0] = 0
    for rep in range(a.reps):
        for label in ("full", "flags_only"):
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.steps):
                ppc.step_1f1b(comm, args[label], s)
            e1.record(s)
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / a.steps], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            res[label].append(t.item())
    assert comm.poll() == 0, comm.error_info()
    ar_per_step = n_ar[0] / (2 * a.reps * a.steps)
    full, ctrl = statistics.median(res["full"]), statistics.median(res["flags_only"])
    layers_all = [None] * world
    dist.all_gather_object(layers_all, layer)
    if rank == 0:
        pp_bytes = 2 * M * nbytes if 0 < stage < S - 1 else M * nbytes   # sent per step
        rec = {"pp": S, "tp": TP, "dp": world // (S * TP), "M": M, "layers_per_stage": per_stage,
               "engine": a.engine, "produce_in_place": a.inplace,
               "ms_step": full, "ms_step_flags_only": ctrl,
               "exposed_frac": (full - ctrl) / full,
               "exposed_frac_per_rep": [(f - c) / f for f, c in zip(res["full"], res["flags_only"])],
               "ms_step_reps": res["full"], "ms_step_flags_only_reps": res["flags_only"],
               "tokens_per_s_per_pipeline": M * T / (full * 1e-3),
               "nccl_tp_allreduces_per_step_per_rank": ar_per_step,
               "egress_per_step_per_gpu": {
                   "pp_bytes_stage0": M * nbytes, "pp_bytes_middle_stage": 2 * M * nbytes,
                   "nccl_allreduce_bytes_per_rank": ar_per_step * nbytes * 2 * (TP - 1) / TP,
                   "note": "ring allreduce sends 2(T-1)/T of the buffer per rank; PP bytes are "
                           "what one stage sends per step"},
               "compute": "LLaMA-8B-shaped MLP GEMMs (h 4096, ffn 14336, split over TP) bf16 via "
                          "cuBLAS, bwd = 2x fwd GEMMs, 2 NCCL TP allreduces per block pass; "
                          "no attention / norms"}
        if a.layer_times:
            rec["layer_ms"] = layers_all
            # NEXT-3: the planner fed with these measured per-layer
            # times — its predicted step time for this split vs the measured one, and the
            # split it recommends for the same total layer count
            from paper_2602_18007_b200.partition import iteration_time, optimize_partition
            by_stage = {}
            for r, lt in enumerate(layers_all):
                by_stage.setdefault(stage_of(r), lt)
            tf = [by_stage[st]["fwd"] for st in range(S)]
            tb = [by_stage[st]["bwd"] for st in range(S)]
            comm_ms = nbytes / (a.comm_gbps * 1e9) * 1e3        # one boundary message
            rec["planner"] = {
                "layers_per_stage": per_stage, "t_fwd_ms": tf, "t_bwd_ms": tb,
                "predicted_ms_step": iteration_time(per_stage, tf, tb, M, comm_ms),
                "measured_ms_step": full,
                "recommended_split": optimize_partition(sum(per_stage), tf, tb, M, comm_ms),
                "ffn_scale_stage0": a.ffn_scale_stage0,
                "model": "paper_2602_18007_b200.partition.iteration_time (1F1B event model, "
                         "per-layer fwd/bwd ms measured alone on each stage)"}
        print(json.dumps(rec), flush=True)
        os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
        with open(a.out, "a") as fh:
            fh.write(json.dumps(rec) + "\n")
    dist.barrier()
    comm.disconnect()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
