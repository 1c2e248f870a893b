"""Throughput of the TP-sliced boundary with the fused all-gather (NEXT-1, ppc_pp_recv_gather)
against the replicated boundary it replaces, PP = 2 x TP = 2 on 4 GPUs (torchrun, one process
per GPU).  Sliced: every TP rank of stage 0 publishes its 1/TP slice (zero-copy); every TP
rank of stage 1 gathers all slices (pulled over NVLink).  Replicated (A17 reading): every
TP rank sends the full tensor to its own peer.  Time = CUDA events on the receivers' stream
over N messages, max over ranks; GB/s per receiver = bytes landed in its buffer / time.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/gather_bench.py [--size 32M]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=32 << 20)
    ap.add_argument("--n", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    tp = 2
    pp_i, tp_i = rank // tp, rank % tp
    total = a.size
    sl = total // tp
    out = {}
    for mode in ("sliced", "replicated"):
        cfg = ppc.make_config(tp=tp, pp=world // tp, dp=1, max_msg_bytes=total,
                              chunk_bytes=256 << 10, zc_async=1)
        comm = ppc.connect_distributed(cfg, rank, world, torch.cuda.current_device(),
                                       with_nccl=False)
        full = torch.empty(total, dtype=torch.uint8, device="cuda")
        ppc.fill_payload(full, total, 42, 0, 0, 0, 0)
        dst = torch.empty(total, dtype=torch.uint8, device="cuda")
        ppc.register_tensors(comm, [full])
        s = torch.cuda.Stream()
        times = []
        mb = 0
        for rep in range(a.reps + 1):
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(a.n):
                if pp_i == 0:
                    if mode == "sliced":
                        comm.send(ppc.FWD, full.data_ptr() + tp_i * sl, sl, mb=mb, stream=s)
                    else:
                        comm.send(ppc.FWD, full, total, mb=mb, stream=s)
                else:
                    if mode == "sliced":
                        comm.recv_gather(ppc.FWD, dst, total, mb=mb, stream=s)
                    else:
                        comm.recv(ppc.FWD, dst, total, mb=mb, stream=s)
                mb += 1
            if pp_i == 0:
                comm.wait_consumed(ppc.FWD, s)
            e1.record(s)
            torch.cuda.synchronize()
            assert comm.poll() == 0, comm.error_info()
            t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            if rep:
                times.append(t.item() * 1e-3)
        ok = True
        if pp_i == 1:
            ok = bool(torch.equal(dst, full))           # every rank filled the same payload
        okt = torch.tensor([0.0 if ok else 1.0])
        dist.all_reduce(okt)
        t = sorted(times)[len(times) // 2]
        out[mode] = {"us_per_msg": t / a.n * 1e6, "gbps_per_receiver": a.n * total / t / 1e9,
                     "nvlink_bytes_per_sender": sl if mode == "sliced" else total,
                     "outputs_ok": okt.item() == 0}
        dist.barrier()
        comm.disconnect()
        dist.barrier()
        comm.destroy()
    if rank == 0:
        print(json.dumps({"pp": world // tp, "tp": tp, "bytes": total, "n": a.n, **out}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
