"""Exposed PP communication in a compute-bearing 1F1B step (BASELINE.json target "exposed PP
communication < 5% of 1F1B step time"; R13 / SURVEY A13).

Stage compute = L LLaMA-8B-shaped MLP blocks per stage on the boundary tensor [4096, 4096]
bf16 (h=4096, ffn=14336: x@W1 -> silu -> @W2; backward runs the same GEMMs twice), cuBLAS via
torch as the *user's model* inside ppc_stage_fn callbacks; the transfers are libppc's.
exposed = (T_step - T_step,flags-only) / T_step, where the flags-only control run uses the same
schedule, streams and flags with zero-byte messages.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 bench_exposure.py --layers 1
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import paper_2602_18007_b200 as ppc  # noqa: E402


class _CAI:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<u2", "data": (ptr, False),
                                         "version": 3, "strides": None}


def as_bf16(ptr, numel):
    return torch.as_tensor(_CAI(ptr, numel), device="cuda").view(torch.bfloat16)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--M", type=int, default=8)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--engine", default="sm")
    ap.add_argument("--out", default="gpurun_out/exposure.jsonl")
    ap.add_argument("--inplace", action="store_true",
                    help="PPC_STEP_INPLACE=1: stage fns produce straight into the peer's slot")
    a = ap.parse_args()
    if a.inplace:
        os.environ["PPC_STEP_INPLACE"] = "1"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    S, M, T, H, F = world, a.M, 4096, 4096, 14336
    nbytes = T * H * 2
    g = torch.Generator(device="cuda").manual_seed(42 + rank)
    W1 = [torch.randn(H, F, device="cuda", dtype=torch.bfloat16, generator=g) * 0.02 for _ in range(a.layers)]
    W2 = [torch.randn(F, H, device="cuda", dtype=torch.bfloat16, generator=g) * 0.02 for _ in range(a.layers)]
    x0 = torch.randn(T, H, device="cuda", dtype=torch.bfloat16, generator=g)

    def compute(inp, out, reps, stream):
        with torch.cuda.stream(torch.cuda.ExternalStream(stream)):
            h = x0 if inp is None else inp.view(T, H)
            for r in range(reps):
                for l in range(a.layers):
                    last = out is not None and r == reps - 1 and l == a.layers - 1
                    # the last GEMM's epilogue stores straight into `out` (with
                    # PPC_STEP_INPLACE: the receiver's ring slot, over NVLink)
                    h = torch.matmul(torch.nn.functional.silu(h @ W1[l]), W2[l],
                                     out=out.view(T, H) if last else None)

    def fwd(user, mb, inp, out, ib, ob, stream):
        compute(as_bf16(inp, T * H) if inp and ib else None, as_bf16(out, T * H) if out and ob else None,
                1, stream)
        return 0

    def bwd(user, mb, inp, out, ib, ob, stream):
        compute(as_bf16(inp, T * H) if inp and ib else None, as_bf16(out, T * H) if out and ob else None,
                2, stream)
        return 0

    eng = {"sm": ppc.ENGINE_SM, "pull": ppc.ENGINE_PULL, "ce": ppc.ENGINE_CE}[a.engine]
    cfg = ppc.make_config(pp=S, max_msg_bytes=nbytes, chunk_bytes=1 << 20, engine=eng)
    comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
    s = torch.cuda.Stream()
    res = {}
    for label, msg in (("full", nbytes), ("flags_only", 0)):
        sa = ppc.StepArgs(M, msg, msg, fwd=fwd, bwd=bwd)
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
        res[label] = t.item()
    assert comm.poll() == 0
    if rank == 0:
        rec = {"pp": S, "M": M, "layers_per_stage": a.layers, "engine": a.engine,
               "produce_in_place": a.inplace,
               "ms_step": res["full"], "ms_step_flags_only": res["flags_only"],
               "exposed_frac": (res["full"] - res["flags_only"]) / res["full"],
               "tokens_per_s": M * T / (res["full"] * 1e-3),
               "compute": "LLaMA-8B-shaped MLP GEMMs (h 4096, ffn 14336) bf16 via cuBLAS, "
                          "bwd = 2x fwd GEMMs; no attention / norms"}
        print(json.dumps(rec), flush=True)
        with open(a.out, "a") as fh:
            fh.write(json.dumps(rec) + "\n")
    dist.barrier()
    comm.disconnect()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
