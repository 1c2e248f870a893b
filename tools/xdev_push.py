"""Single-process NVLink push/recv measurement: two virtual stages on cuda:0 and cuda:1,
ordered by CUDA events (no cross-process spins), so the push kernel can be profiled with
ncu replay safely.  Prints per-launch device times of push and recv kernels.

    python tools/xdev_push.py --size 32M --n 40 [--cta 32 --chunk 1M --mode uni|bidir]
"""
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


ap = argparse.ArgumentParser()
ap.add_argument("--size", default="32M")
ap.add_argument("--n", type=int, default=40)
ap.add_argument("--cta", type=int, default=32)
ap.add_argument("--chunk", default="1M")
ap.add_argument("--mode", default="uni")
ap.add_argument("--engine", default="sm")
ap.add_argument("--channels", type=int, default=1)
a = ap.parse_args()
n = size_of(a.size)
cfg = ppc.make_config(pp=2, max_msg_bytes=n, chunk_bytes=size_of(a.chunk), cta_per_channel=a.cta,
                      engine={"sm": ppc.ENGINE_SM, "ce": ppc.ENGINE_CE, "pull": ppc.ENGINE_PULL}[a.engine],
                      channels=a.channels, trace=2)
comms = ppc.virtual_stages(cfg, [0, 1])
src = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
dst = [torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
for d in (0, 1):
    with torch.cuda.device(d):
        ppc.fill_payload(src[d], n, 42, 0, 0, d, 0)
ss = [torch.cuda.Stream(device=d) for d in (0, 1)]
rs = [torch.cuda.Stream(device=d) for d in (0, 1)]


def run(N):
    for i in range(N):
        comms[0].send(ppc.FWD, src[0], n, mb=i, stream=ss[0])
        if a.mode == "bidir":
            comms[1].send(ppc.BWD, src[1], n, mb=i, stream=ss[1])
        comms[1].recv(ppc.FWD, dst[1], n, mb=i, stream=rs[1])
        if a.mode == "bidir":
            comms[0].recv(ppc.BWD, dst[0], n, mb=i, stream=rs[0])
    for d in (0, 1):
        torch.cuda.synchronize(d)


run(4)
for c in comms:
    c.kernel_times(0), c.kernel_times(1)
run(a.n)
push = comms[0].kernel_times(0)
recv = comms[1].kernel_times(1)
assert torch.equal(dst[1].cpu(), src[0].cpu())
out = {"size": n, "n": a.n, "mode": a.mode, "cta": a.cta, "chunk": a.chunk, "engine": a.engine,
       "push_us_median": statistics.median(push) * 1e3,
       "push_gbps_median": n / (statistics.median(push) * 1e-3) / 1e9,
       "push_gbps_best": n / (min(push) * 1e-3) / 1e9,
       "recv_us_median": statistics.median(recv) * 1e3}
print(json.dumps(out))
for c in comms:
    assert c.poll() == 0
    c.disconnect()
for c in comms:
    c.destroy()
