"""Litmus stress of the transfer protocol: >= 10^6 messages of random sizes
and offsets, both directions at once, K = 2 ring slots (every slot reused ~500k times),
4 KiB chunks (multi-chunk messages, ragged tails, misaligned sources and destinations),
over the cross-process protocol on one GPU (cfg.local_spin: device flag / credit / header
spins with .sys scope) — ring push, or zero-copy pulls from a registered buffer — with
plain and batched receives mixed at random.  Every received byte is compared on the device
with the bytes the sender sent (one big source buffer per direction, message i = a random
slice of it; the receiver writes message i at its own offset of a receive log).

    python tools/litmus.py --messages 1000000 [--zc] [--seed 1]

Prints one JSON line: messages, bytes, mismatching bytes, latched errors, seconds."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--messages", type=int, default=1_000_000, help="total over both directions")
    ap.add_argument("--max-bytes", type=int, default=8192)
    ap.add_argument("--chunk", type=int, default=4096)
    ap.add_argument("--K", type=int, default=2)
    ap.add_argument("--zc", action="store_true")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    per_dir = a.messages // 2
    src_bytes = 64 << 20
    cfg = ppc.make_config(pp=2, max_msg_bytes=a.max_bytes, chunk_bytes=a.chunk, ring_slots=a.K,
                          local_spin=1, timeout_ns=5_000_000_000)
    comms = ppc.local_comms(cfg, 0)
    src = [torch.empty(src_bytes, dtype=torch.uint8, device="cuda") for _ in range(2)]
    for d in (0, 1):
        ppc.fill_payload(src[d], src_bytes, 42, 0, 0, d, 0)
    if a.zc:
        ppc.register_local(comms, [[src[0]], [src[1]]])
    sizes = [rng.integers(0, a.max_bytes + 1, per_dir) for _ in range(2)]
    offs = [rng.integers(0, src_bytes - a.max_bytes, per_dir) for _ in range(2)]
    cum = [np.concatenate([[0], np.cumsum(sz)]) for sz in sizes]
    logs = [torch.zeros(int(c[-1]) + 64, dtype=torch.uint8, device="cuda") for c in cum]
    st = [torch.cuda.Stream() for _ in range(4)]        # send FWD, recv FWD, send BWD, recv BWD
    sb = [src[d].data_ptr() for d in (0, 1)]
    lb = [logs[d].data_ptr() for d in (0, 1)]
    t0 = time.perf_counter()
    i = [0, 0]
    while i[0] < per_dir or i[1] < per_dir:
        for d in (0, 1):
            if i[d] >= per_dir:
                continue
            snd, rcv = (0, 1) if d == 0 else (1, 0)
            k = 1 if rng.random() < 0.5 else int(min(rng.integers(2, 9), per_dir - i[d]))
            # a batch may span more than K messages: its later sends wait (on the device) for
            # the credits the same batch returns mid-way
            for j in range(i[d], i[d] + k):
                comms[snd].send(d, sb[d] + int(offs[d][j]), int(sizes[d][j]), mb=j,
                                stream=st[2 * d])
            if k == 1:
                comms[rcv].recv(d, lb[d] + int(cum[d][i[d]]), int(sizes[d][i[d]]), mb=i[d],
                                stream=st[2 * d + 1])
            else:
                comms[rcv].recv_batch(d, [lb[d] + int(cum[d][j]) for j in range(i[d], i[d] + k)],
                                      [int(sizes[d][j]) for j in range(i[d], i[d] + k)],
                                      mb0=i[d], stream=st[2 * d + 1])
            i[d] += k
    torch.cuda.synchronize()
    t_run = time.perf_counter() - t0
    errors = [ppc.STATUS[c.poll()] for c in comms if c.poll()]
    # device-side verification, at most 20k messages / 512 MiB at a time (the gather index
    # tensors stay far below 2^31 elements): gather the expected bytes
    bad = 0
    for d in (0, 1):
        a0 = 0
        while a0 < per_dir:
            a1 = min(per_dir, a0 + 20_000,
                     int(np.searchsorted(cum[d], cum[d][a0] + (512 << 20), side="right")) - 1)
            lo, a0 = a0, max(a1, a0 + 1)
            sz = torch.from_numpy(sizes[d][lo:a0]).cuda()
            of = torch.from_numpy(offs[d][lo:a0]).cuda()
            tot = int(sz.sum())
            if tot == 0:
                continue
            starts = torch.repeat_interleave(of, sz)
            first = torch.cumsum(sz, 0) - sz
            within = torch.arange(tot, device="cuda") - torch.repeat_interleave(first, sz)
            want = src[d][starts + within]
            got = logs[d][int(cum[d][lo]):int(cum[d][lo]) + tot]
            bad += int((want != got).sum())
    rec = {"messages": 2 * per_dir, "bytes": int(sum(c[-1] for c in cum)), "zero_copy": a.zc,
           "K": a.K, "chunk": a.chunk, "max_bytes": a.max_bytes, "mismatching_bytes": bad,
           "errors": errors, "seconds": t_run, "seed": a.seed,
           "mode": "cfg.local_spin on one GPU, both directions, plain + batched receives"}
    print(json.dumps(rec), flush=True)
    if a.out:
        with open(a.out, "a") as fh:
            fh.write(json.dumps(rec) + "\n")
    for c in comms:
        c.disconnect()
    for c in comms:
        c.destroy()
    assert bad == 0 and not errors


if __name__ == "__main__":
    main()
