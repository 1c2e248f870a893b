"""Small one-GPU workload for compute-sanitizer (memcheck / racecheck / synccheck):
    python tools/sanitize_smoke.py [--spin] && compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
Covers the ring push/recv (SM, CE, PULL engines, misaligned and ragged sizes), the batched
receive, the direct single-copy step, a CUDA-graph replay and the XOR stage kernels, checked
against synth.  --spin adds smoke()'s cross-process-protocol paths (device-spin ring and
zero-copy with fused publication on one GPU), which need the sender's and the receiver's
kernels to run concurrently (a tool that serialises kernels turns them into TIMEOUTs)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import __graft_entry__  # noqa: E402
import paper_2602_18007_b200 as ppc  # noqa: E402
from synth import payload as P  # noqa: E402


def main():
    if "--spin" in sys.argv:
        __graft_entry__.smoke()
    s = torch.cuda.current_stream()
    for eng in (ppc.ENGINE_SM, ppc.ENGINE_CE, ppc.ENGINE_PULL):
        comms = ppc.virtual_stages(ppc.make_config(pp=2, max_msg_bytes=1 << 20, chunk_bytes=64 << 10,
                                                   engine=eng), 0)
        for i, (n, off) in enumerate([(1, 1), (33, 0), (3 * (64 << 10) + 5, 3), ((1 << 20) - 64, 16)]):
            src = torch.empty(n + 64, dtype=torch.uint8, device="cuda")
            dst = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
            ppc.fill_payload(src.data_ptr() + off, n, 42, 0, 0, 0, i)
            comms[0].send(ppc.FWD, src.data_ptr() + off, n, mb=i, stream=s)
            comms[1].recv(ppc.FWD, dst.data_ptr() + off, n, mb=i, stream=s)
            torch.cuda.synchronize()
            assert np.array_equal(dst.cpu().numpy()[off:off + n], P.payload_bytes(42, 0, 0, 0, i, n))
        sizes = [5, 3 * (64 << 10) + 7, 64 << 10]
        outs = [torch.zeros(n, dtype=torch.uint8, device="cuda") for n in sizes]
        srcs = []
        for i, n in enumerate(sizes):
            b = torch.empty(n, dtype=torch.uint8, device="cuda")
            srcs.append(b)
            ppc.fill_payload(b, n, 42, 0, 0, 0, 10 + i)
            comms[0].send(ppc.FWD, b, n, mb=10 + i, stream=s)
        comms[1].recv_batch(ppc.FWD, outs, sizes, mb0=10, stream=s)      # batched receive
        torch.cuda.synchronize()
        for i, n in enumerate(sizes):
            assert np.array_equal(outs[i].cpu().numpy(), P.payload_bytes(42, 0, 0, 0, 10 + i, n))
        for c in comms:
            assert c.poll() == 0
            c.disconnect()
        for c in comms:
            c.destroy()
    for direct in ("1", "0"):
        os.environ["PPC_LOCAL_DIRECT"] = direct
        S, M, n = 3, 4, 2 * (64 << 10) + 17
        comms = ppc.virtual_stages(ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=64 << 10), 0)
        bufs = lambda: [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
        X, G, Y, DX = bufs(), bufs(), bufs(), bufs()
        for m in range(M):
            ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
            ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
        args = [ppc.StepArgs(M, n, n, x=X if k == 0 else None, g=G if k == S - 1 else None,
                             y=Y if k == S - 1 else None, dx=DX if k == 0 else None) for k in range(S)]
        streams = [torch.cuda.Stream() for _ in range(S)]
        ppc.step_1f1b_local(comms, args, streams)
        g = ppc.StepGraph(comms, args, streams)
        g.launch()
        torch.cuda.synchronize()
        for m in range(M):
            assert torch.equal(Y[m], X[m]) and torch.equal(DX[m], G[m])
        g.destroy()
        for c in comms:
            assert c.poll() == 0
            c.disconnect()
        for c in comms:
            c.destroy()
    print("sanitize_smoke OK", flush=True)


if __name__ == "__main__":
    main()
