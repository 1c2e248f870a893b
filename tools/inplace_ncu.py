"""One-process target for ncu of the fused produce-in-place kernel (xor_send_kernel): two
virtual stages on GPU 0 and GPU 1 (ordered by CUDA events, no device spins, so ncu's kernel
replay cannot deadlock); stage 0 computes the XOR proxy of a 32 MiB boundary tensor straight
into stage 1's ring slot over NVLink, stage 1 receives.  Checks the bytes at the end.

    ncu --set full -k regex:xor_send_kernel -s 2 -c 1 python tools/inplace_ncu.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2602_18007_b200 as ppc  # noqa: E402
from synth import payload as P  # noqa: E402


def main():
    n, M = 32 << 20, int(os.environ.get("M", "6"))
    cfg = ppc.make_config(pp=2, max_msg_bytes=n, chunk_bytes=256 << 10)
    comms = ppc.virtual_stages(cfg, [0, 1])
    x = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    y = torch.empty(n, dtype=torch.uint8, device="cuda:1")
    s0, s1 = torch.cuda.Stream(device=0), torch.cuda.Stream(device=1)
    for m in range(M):
        ppc.fill_payload(x, n, 42, 0, 0, 0, m, stream=s0)
        comms[0].xor_send(ppc.FWD, ppc.XorCtx(42, 0, 0, 0), m, x, n, stream=s0)
        comms[1].recv(ppc.FWD, y, n, mb=m, stream=s1)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    want = P.payload_bytes(42, 0, 0, 0, M - 1, n) ^ P.proxy_mask(42, 0, 0, 0, M - 1, n)
    assert np.array_equal(y.cpu().numpy(), want)
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()
    print("inplace_ncu OK")


if __name__ == "__main__":
    main()
