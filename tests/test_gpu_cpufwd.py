"""Path equivalence: the CPU-Forwarding baseline B1 (libppcb:
D2H -> pinned /dev/shm ring -> H2D) and the device-direct path (libppc) deliver the same
messages — the delivery log (seq, mb, bytes, blake2b-128 digest) of every (boundary,
direction) is identical for both and equal to the CPU oracle's (oracle/transfer.py via
oracle/proxy.run_1f1b) on the same seeded inputs, and the delivered bytes are identical."""
import os

import numpy as np
import pytest
import torch

import paper_2602_18007_b200 as ppc
from oracle.proxy import run_1f1b
from oracle.transfer import digest
from paper_2602_18007_b200.cpufwd import CpuFwdLink
from synth import payload as P

pytestmark = pytest.mark.gpu


def _b1_step(X, G, n, M, K, channels, chunk, tag):
    """One comm-only 1F1B step of a PP = 2 pipeline over B1, both stages in this process,
    stepped by one host thread in dependency order (a send never blocks on a full ring)."""
    s = torch.cuda.current_stream()
    # one shared ring per direction: the sender end creates "/ppcb_<dir>_<tag>", the
    # receiver end opens the same name
    links = {name: CpuFwdLink(f"{name[0]}_{tag}_{os.getpid()}", snd, n, chunk, K, channels, 0)
             for name, snd in (("fs", True), ("fr", False), ("bs", True), ("br", False))}
    for ln in links.values():
        ln.connect()
    Y = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
    DX = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
    ops = [ppc.schedule_1f1b(2, st, M) for st in (0, 1)]
    i, sent, recvd = [0, 0], [0, 0], [0, 0]
    log = {0: [], 1: []}
    while i[0] < len(ops[0]) or i[1] < len(ops[1]):
        prog = False
        for st in (0, 1):
            if i[st] >= len(ops[st]):
                continue
            kind, m = ops[st][i[st]]
            d = 0 if kind == "F" else 1
            if (st == 0) == (d == 0):                     # this op sends
                if sent[d] - recvd[d] >= K:
                    continue
                (links["fs"].send(X[m], n, m, s) if d == 0 else links["bs"].send(G[m], n, m, s))
                sent[d] += 1
            else:
                if recvd[d] >= sent[d]:
                    continue
                out = Y[m] if d == 0 else DX[m]
                (links["fr"] if d == 0 else links["br"]).recv(out, n, m, s)
                recvd[d] += 1
                torch.cuda.synchronize()
                log[d].append((recvd[d], m, n, digest(out.cpu().numpy())))
            i[st] += 1
            prog = True
        assert prog
    for ln in links.values():
        ln.destroy()
    return Y, DX, log


@pytest.mark.parametrize("n,chunk,channels", [(131072, 64 << 10, 1),          # C1 boundary
                                              (3 * 65536 + 1234, 64 << 10, 4),  # ragged tail
                                              (5, 4096, 2)])
def test_b1_and_device_direct_logs_identical(n, chunk, channels, monkeypatch):
    M, K = 6, 2
    xs = [P.source_activation(42, 0, m, n) for m in range(M)]
    gs = [P.source_gradient(42, 0, m, n) for m in range(M)]
    ident = lambda s_, m, x: x
    Yo, DXo, chans, _ = run_1f1b(2, M, K, ident, ident, lambda m: xs[m], lambda m: gs[m], n, n, n)
    olog = {d: chans[(d, 0)].log for d in (0, 1)}
    X = [torch.from_numpy(x.copy()).cuda() for x in xs]
    G = [torch.from_numpy(g.copy()).cuda() for g in gs]
    torch.cuda.synchronize()
    # CPU-Forwarding B1
    Yb, DXb, blog = _b1_step(X, G, n, M, K, channels, chunk, f"{n}_{channels}")
    # device-direct, ring path of virtual stages (push -> chunk flags -> copy-out), traced
    monkeypatch.setenv("PPC_LOCAL_DIRECT", "0")
    cfg = ppc.make_config(pp=2, max_msg_bytes=n, ring_slots=K, chunk_bytes=max(chunk, 4096),
                          trace=1)
    comms = ppc.virtual_stages(cfg, 0)
    Yd = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
    DXd = [torch.zeros(n, dtype=torch.uint8, device="cuda") for _ in range(M)]
    args = [ppc.StepArgs(M, n, n, x=X, dx=DXd), ppc.StepArgs(M, n, n, g=G, y=Yd)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    ppc.step_1f1b_local(comms, args, streams)
    torch.cuda.synchronize()
    dlog = {0: [], 1: []}
    for c, d, outs in ((comms[1], 0, Yd), (comms[0], 1, DXd)):
        recs = [r for r in c.trace() if r["kind"] == 1]
        for r in recs:
            dlog[d].append((r["seq"], r["mb"], r["bytes"], digest(outs[r["mb"]].cpu().numpy())))
    for cm in comms:
        assert cm.poll() == 0
        cm.disconnect()
    for cm in comms:
        cm.destroy()
    for d in (0, 1):
        assert blog[d] == olog[d], d                     # B1 log == oracle log
        assert dlog[d] == olog[d], d                     # device-direct log == oracle log
    for m in range(M):
        for got in (Yb[m], Yd[m]):
            assert np.array_equal(got.cpu().numpy(), Yo[m]), m
        for got in (DXb[m], DXd[m]):
            assert np.array_equal(got.cpu().numpy(), DXo[m]), m
