"""Produce-in-place sends vs compute-then-send on 2 GPUs (torchrun --nproc-per-node 2).

Rank 0 runs the XOR stage proxy on a 32 MiB boundary tensor and sends it to rank 1, M
messages back to back; rank 1 receives into its user buffer.  Variants:
  classic   ppc_stage_xor into a local buffer, then ppc_pp_send (SM push, or a zero-copy
            publication of a registered buffer: classic_zc)
  inplace   ppc_pp_send_begin, ppc_stage_xor writing into the peer slot, ppc_pp_send_end
  fused     ppc_pp_send_begin, ppc_stage_xor_send (per-chunk flags from the producer), end
One JSON line per variant: us per message on the receiver's stream (CUDA events around the
M messages, after warm-up), max over the two ranks."""
import argparse
import ctypes as C
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=32 << 20)
    ap.add_argument("--M", type=int, default=16)
    ap.add_argument("--chunk", type=int, default=512 << 10)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--variants", default="classic,classic_zc,inplace,fused")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo")
    n = args.bytes
    cfg = ppc.make_config(pp=2, max_msg_bytes=n, chunk_bytes=args.chunk)
    comm = ppc.connect_distributed(cfg, rank, world, rank, with_nccl=False)
    s = torch.cuda.Stream()
    xor = ppc._lib.ppc_stage_xor
    xor.restype = C.c_int
    xor.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t,
                    C.c_void_p]
    ctx = ppc.XorCtx(42, 0, 0, 0)
    x = torch.empty(n, dtype=torch.uint8, device="cuda")
    ppc.fill_payload(x, n, 42, 0, 0, 0, 0)
    y = torch.empty(n, dtype=torch.uint8, device="cuda")
    blob = comm.register(y)
    blobs = [None] * world
    dist.all_gather_object(blobs, blob)
    for b in blobs:
        comm.register_import(b)
    torch.cuda.synchronize()

    def one(variant, m):
        if rank == 1:
            comm.recv(ppc.FWD, y, n, mb=m, stream=s)
            return
        if variant.startswith("classic"):
            out = y if variant == "classic_zc" else x2
            assert xor(C.byref(ctx), m, x.data_ptr(), out.data_ptr(), n, n, s.cuda_stream) == 0
            comm.send(ppc.FWD, out, n, mb=m, stream=s)
        elif variant == "inplace":
            sl = comm.send_begin(ppc.FWD, n, m, stream=s)
            assert xor(C.byref(ctx), m, x.data_ptr(), sl.payload, n, n, s.cuda_stream) == 0
            comm.send_end(ppc.FWD, False, stream=s)
        else:
            comm.xor_send(ppc.FWD, ctx, m, x, n, stream=s)

    x2 = torch.empty(n, dtype=torch.uint8, device="cuda")   # unregistered: ring push
    mb = 0
    for variant in args.variants.split(","):
        times = []
        for rep in range(args.reps + 1):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(args.M):
                one(variant, mb)
                mb += 1
            e1.record(s)
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1) * 1e3 / args.M)
        t = torch.tensor([min(times), sorted(times)[len(times) // 2]], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"variant": variant, "bytes": n, "M": args.M, "chunk": args.chunk,
                              "us_per_msg_best": t[0].item(), "us_per_msg_median": t[1].item(),
                              "gbps_median": n / (t[1].item() * 1e-6) / 1e9}), flush=True)
    assert comm.poll() == 0, ppc.STATUS[comm.poll()]
    dist.barrier()
    comm.disconnect()
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
