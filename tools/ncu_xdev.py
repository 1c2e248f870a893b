"""Cross-GPU transfer kernels in ONE process, so ncu can profile them with NVLink counters
(a multi-rank torchrun command is never run under ncu): stage 0 on cuda:0, stage 1 on cuda:1,
cfg.local_spin (the cross-process protocol: device flags, zero-copy publication).  The host
enqueues every send before its receive and the zero-copy sends complete at publication
(cfg.zc_async), so ncu's kernel serialisation never leaves a kernel waiting for one that has
not run yet.

    python tools/ncu_xdev.py --mode zc|push [--size 32M --n 4]
    ncu --metrics gpu__time_duration.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,\\
        dram__bytes_read.sum,dram__bytes_write.sum -k regex:recv_kernel python tools/ncu_xdev.py

Without ncu it prints the per-launch event times of the receive (zc) or push kernels."""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402


def size_of(s):
    u = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    return int(s[:-1]) * u[s[-1]] if s[-1] in u else int(s)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="zc", choices=["zc", "push"])
    ap.add_argument("--size", default="32M")
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--chunk", default="256K")
    a = ap.parse_args()
    n = size_of(a.size)
    cfg = ppc.make_config(pp=2, max_msg_bytes=n, chunk_bytes=size_of(a.chunk), local_spin=1,
                          zc_async=1, ring_slots=a.n + 1, trace=2)
    comms = ppc.local_comms(cfg, [0, 1])
    src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    dst = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    with torch.cuda.device(0):
        ppc.fill_payload(src, n, 42, 0, 0, 0, 0)
    torch.cuda.synchronize(0)
    if a.mode == "zc":
        ppc.register_local(comms, [[src], []])
    s0 = torch.cuda.Stream(device=0)
    s1 = torch.cuda.Stream(device=1)
    for i in range(a.n):
        comms[0].send(ppc.FWD, src, n, mb=i, stream=s0)
        comms[1].recv(ppc.FWD, dst, n, mb=i, stream=s1)
    comms[0].wait_consumed(ppc.FWD, s0)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    ok = torch.equal(dst.cpu(), src.cpu())
    k = comms[1].kernel_times(1) if a.mode == "zc" else comms[0].kernel_times(0)
    print(json.dumps({"mode": a.mode, "bytes": n, "n": a.n, "outputs_ok": ok,
                      "kernel_us_median": statistics.median(k) * 1e3 if k else None,
                      "errors": [c.error_info() for c in comms]}), flush=True)
    for c in comms:
        c.disconnect()
    for c in comms:
        c.destroy()
    assert ok


if __name__ == "__main__":
    main()
