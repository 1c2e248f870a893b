"""GPU parity of the transfer path on one B200: virtual stages of one pipeline in one
process (the intra-device ring, K11), through the C-ABI.  Every comparison is element by
element against the oracle (oracle/transfer.py, oracle/proxy.py) on the same seeded
inputs (synth/payload.py), bit-exact."""
import ctypes as C
import hashlib

import numpy as np
import pytest
import torch

import paper_2602_18007_b200 as ppc
from oracle.proxy import run_1f1b, xor_closed_form, xor_stage
from synth import payload as P

pytestmark = pytest.mark.gpu

DEV = 0


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint8).reshape(-1)


def _buf(n):
    return torch.empty(max(n, 1), dtype=torch.uint8, device=f"cuda:{DEV}")


@pytest.mark.parametrize("n", [1, 7, 8, 13, 4096 + 5, (1 << 20) + 3, 32 << 20])
def test_fill_matches_synth(n):
    b = _buf(n)
    ppc.fill_payload(b, n, seed=42, step=1, boundary=2, direction=1, mb=7)
    assert np.array_equal(_host(b)[:n], P.payload_bytes(42, 1, 2, 1, 7, n))


def _pair(**kw):
    cfg = ppc.make_config(pp=kw.pop("pp", 2), **kw)
    return ppc.virtual_stages(cfg, DEV)


@pytest.mark.parametrize("K", [1, 2, 3])
@pytest.mark.parametrize("sizes", [[0, 1, 100, 65536, 3 * 65536 + 17, (5 << 20) + 3, 4096]])
def test_send_recv_bit_exact(K, sizes):
    comms = _pair(max_msg_bytes=8 << 20, ring_slots=K, chunk_bytes=64 << 10)
    s = torch.cuda.current_stream()
    for i, n in enumerate(sizes * 2):              # more messages than slots: ring wraps
        for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
            src = _buf(n)
            ppc.fill_payload(src, n, seed=42, step=0, boundary=0, direction=d, mb=i)
            dst = _buf(n)
            dst.fill_(0xAB)
            comms[snd].send(d, src, n, mb=i, stream=s)
            comms[rcv].recv(d, dst, n, mb=i, stream=s)
            assert np.array_equal(_host(dst)[:n], P.payload_bytes(42, 0, 0, d, i, n)), (i, n, d)
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("n", [5, 4096 + 3, 3 * (64 << 10) + 1234])
@pytest.mark.parametrize("K", [1, 2])
def test_produce_in_place_send(K, n, fused):
    """ppc_pp_send_begin / _end: the producer writes straight into the receiver's ring slot.
    fused: the XOR stage proxy releases each chunk's flag itself (ppc_stage_xor_send);
    otherwise a plain producer (the payload fill, written into the slot) and send_end
    releases the flags.  Both directions, more messages than slots, bit-exact vs the
    oracle's payload / mask streams."""
    comms = _pair(max_msg_bytes=n, ring_slots=K, chunk_bytes=64 << 10)
    s = torch.cuda.current_stream()
    for m in range(4):
        for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
            dst = _buf(n)
            dst.fill_(0xAB)
            want = P.payload_bytes(42, 0, 0, d, m, n)
            if fused:
                src = _buf(n)
                ppc.fill_payload(src, n, 42, 0, 0, d, m, stream=s)
                comms[snd].xor_send(d, ppc.XorCtx(42, 0, snd, d), m, src, n, stream=s)
                want = want ^ P.proxy_mask(42, 0, snd, d, m, n)
            else:
                sl = comms[snd].send_begin(d, n, m, stream=s)
                assert sl.bytes == n and sl.seq == m + 1
                ppc.fill_payload(sl.payload, n, 42, 0, 0, d, m, stream=s)
                comms[snd].send_end(d, False, stream=s)
            comms[rcv].recv(d, dst, n, mb=m, stream=s)
            assert np.array_equal(_host(dst)[:n], want), (m, d)
    # state errors: second begin, a plain send while a slot is open, end without begin
    sl = comms[0].send_begin(ppc.FWD, n, 4, stream=s)
    st = ppc.STATUS.index("STATE")
    assert ppc._send_begin(comms[0].h, ppc.FWD, n, 5, None, C.byref(ppc.Slot())) == st
    assert comms[0].pp_send(ppc.FWD, _buf(n), n, 5, s) == st
    assert ppc._send_end(comms[0].h, ppc.BWD, 0, None) == st
    ppc.fill_payload(sl.payload, n, 42, 0, 0, 0, 4, stream=s)
    comms[0].send_end(ppc.FWD, False, stream=s)
    dst = _buf(n)
    comms[1].recv(ppc.FWD, dst, n, mb=4, stream=s)
    assert np.array_equal(_host(dst)[:n], P.payload_bytes(42, 0, 0, 0, 4, n))
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("engine", [ppc.ENGINE_SM, ppc.ENGINE_CE, ppc.ENGINE_PULL])
@pytest.mark.parametrize("src_off,dst_off", [(1, 0), (0, 3), (8, 8), (16, 48)])
def test_misaligned_buffers(engine, src_off, dst_off):
    """User buffers at byte offsets (16-B vector path, 32-B path, byte fallback) stay exact."""
    comms = _pair(max_msg_bytes=1 << 20, chunk_bytes=64 << 10, engine=engine)
    s = torch.cuda.current_stream()
    for i, n in enumerate([1, 33, 3 * (64 << 10) + 5, (1 << 20) - 64]):
        src = _buf(n + 64)
        dst = _buf(n + 64)
        dst.fill_(0xCD)
        ppc.fill_payload(src.data_ptr() + src_off, n, 42, 0, 0, 0, i)
        comms[0].send(ppc.FWD, src.data_ptr() + src_off, n, mb=i, stream=s)
        comms[1].recv(ppc.FWD, dst.data_ptr() + dst_off, n, mb=i, stream=s)
        got = _host(dst)
        assert np.array_equal(got[dst_off:dst_off + n], P.payload_bytes(42, 0, 0, 0, i, n))
        assert (got[:dst_off] == 0xCD).all() and (got[dst_off + n:] == 0xCD).all()   # no overrun
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()


def test_would_block_and_header_errors():
    comms = _pair(max_msg_bytes=1 << 20, ring_slots=2, chunk_bytes=64 << 10)
    s = torch.cuda.current_stream()
    src, dst = _buf(4096), _buf(4096)
    assert comms[1].pp_recv(ppc.FWD, dst, 4096, 0, s) == ppc.WOULD_BLOCK   # nothing sent
    for m in range(2):
        comms[0].send(ppc.FWD, src, 4096, mb=m, stream=s)
    assert comms[0].pp_send(ppc.FWD, src, 4096, 2, s) == ppc.WOULD_BLOCK    # both slots full
    comms[1].recv(ppc.FWD, dst, 4096, mb=0, stream=s)
    comms[1].recv(ppc.FWD, dst, 2048, mb=1, stream=s)                        # wrong size
    torch.cuda.synchronize()
    assert ppc.STATUS[comms[1].poll()] == "SIZE_MISMATCH"
    assert comms[1].pp_recv(ppc.FWD, dst, 4096, 2, s) == ppc.STATUS.index("STATE")   # poisoned
    for c in comms:
        c.disconnect()
    for c in comms:
        c.destroy()
    comms = _pair(max_msg_bytes=1 << 20)
    comms[0].send(ppc.FWD, src, 4096, mb=3, stream=s)
    comms[1].recv(ppc.FWD, dst, 4096, mb=4, stream=s)                         # wrong mb
    torch.cuda.synchronize()
    assert ppc.STATUS[comms[1].poll()] == "ORDER"
    for c in comms:
        c.disconnect()
    for c in comms:
        c.destroy()


def _masks(n):
    cache = {}

    def mask(s, d, m):
        if (s, d, m) not in cache:
            cache[(s, d, m)] = P.proxy_mask(42, 0, s, d, m, n)
        return cache[(s, d, m)]
    return mask


def _xor_step(S, M, n, K=2, chunk=64 << 10, engine=ppc.ENGINE_SM, trace=0):
    cfg = ppc.make_config(pp=S, max_msg_bytes=max(n, 1), ring_slots=K, chunk_bytes=chunk,
                          engine=engine, trace=trace, channels=2 if engine else 1)
    comms = ppc.virtual_stages(cfg, DEV)
    X = [_buf(n) for _ in range(M)]
    G = [_buf(n) for _ in range(M)]
    Y = [_buf(n) for _ in range(M)]
    DX = [_buf(n) for _ in range(M)]
    for m in range(M):
        ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    torch.cuda.synchronize()        # inputs (legacy stream) before the stage streams
    ctx = [(ppc.XorCtx(42, 0, s, 0), ppc.XorCtx(42, 0, s, 1)) for s in range(S)]
    args = [ppc.StepArgs(M, n, n, fwd=ppc.STAGE_XOR, bwd=ppc.STAGE_XOR, fwd_user=ctx[s][0],
                         bwd_user=ctx[s][1], x=X if s == 0 else None, g=G if s == S - 1 else None,
                         y=Y if s == S - 1 else None, dx=DX if s == 0 else None)
            for s in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    ppc.step_1f1b_local(comms, args, streams)
    torch.cuda.synchronize()
    return comms, Y, DX


@pytest.mark.parametrize("S,M", [(2, 1), (2, 4), (3, 4), (4, 8), (5, 3)])
@pytest.mark.parametrize("engine,direct", [(ppc.ENGINE_SM, 0), (ppc.ENGINE_CE, 0),
                                           (ppc.ENGINE_PULL, 0), (ppc.ENGINE_SM, 1)])
def test_xor_1f1b_step_matches_oracle(S, M, engine, direct, monkeypatch):
    """direct=0: the ring path (push -> flags -> copy-out) of each engine; direct=1: the
    single-copy hand-off of same-GPU virtual stages (no engine involved)."""
    monkeypatch.setenv("PPC_LOCAL_DIRECT", str(direct))
    n = 3 * (64 << 10) + 1234                          # several chunks + ragged tail
    comms, Y, DX = _xor_step(S, M, n, engine=engine, trace=1)
    mask = _masks(n)
    src = lambda m: P.source_activation(42, 0, m, n)
    dsrc = lambda m: P.source_gradient(42, 0, m, n)
    Yo, DXo, chans, _ = run_1f1b(S, M, 2, xor_stage(mask, 0), xor_stage(mask, 1), src, dsrc,
                                 n, n, n)
    for m in range(M):
        assert np.array_equal(_host(Y[m])[:n], Yo[m]), m
        assert np.array_equal(_host(DX[m])[:n], DXo[m]), m
        y, g = xor_closed_form(S, m, src(m), dsrc(m), mask)
        assert np.array_equal(Yo[m], y) and np.array_equal(DXo[m], g)
    # exactly once, in order: every receive record of every stage in ascending seq / mb
    for c in comms:
        assert c.poll() == 0
        if direct:
            continue
        recs = [r for r in c.trace() if r["kind"] == 1]
        for d in (0, 1):
            rs = [r for r in recs if r["src"] == (c.rank - 1 if d == 0 else c.rank + 1)]
            assert [r["seq"] for r in rs] == list(range(1, len(rs) + 1))
            assert [r["mb"] for r in rs] == list(range(len(rs)))
            assert all(r["t_end_ns"] >= r["t_start_ns"] > 0 for r in rs)
    for c in comms:
        c.disconnect()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("tma_ctas", [148, 7, 0])
@pytest.mark.parametrize("n", [5, 16, 4096 + 3, 3 * (64 << 10) + 1234, (5 << 20) + 7])
def test_direct_copy_engines(n, tma_ctas, monkeypatch):
    """The virtual-stage hand-off copy (K11) in both engines: TMA bulk (148 CTAs, and 7 so
    every CTA walks many tiles around its 6-stage ring) and SIMT (0, the default); sizes below one 16-B
    bulk unit, exactly one, a partial tile, several tiles with a ragged tail, and more
    tiles than CTAs.  Output bit-exact against the oracle's 1F1B simulation."""
    monkeypatch.setenv("PPC_LOCAL_DIRECT", "1")
    monkeypatch.setenv("PPC_COPY_TMA_CTAS", str(tma_ctas))
    S, M = 3, 4
    comms, Y, DX = _xor_step(S, M, n)
    mask = _masks(n)
    Yo, DXo, _, _ = run_1f1b(S, M, 2, xor_stage(mask, 0), xor_stage(mask, 1),
                             lambda m: P.source_activation(42, 0, m, n),
                             lambda m: P.source_gradient(42, 0, m, n), n, n, n)
    for m in range(M):
        assert np.array_equal(_host(Y[m])[:n], Yo[m]), m
        assert np.array_equal(_host(DX[m])[:n], DXo[m]), m
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("K", [1, 2])
@pytest.mark.parametrize("S,M", [(2, 1), (2, 4), (3, 4), (4, 8)])
def test_xor_step_produce_in_place(S, M, K, monkeypatch):
    """PPC_STEP_INPLACE=1: in the 1F1B step every stage fn whose output is sent writes it
    straight into the receiver's ring slot (ppc_pp_send_begin / _end on the compute stream;
    the sender blocks on a full ring as in the oracle's event model, A4).  Virtual stages,
    ring path; outputs bit-exact vs the oracle's 1F1B simulation."""
    monkeypatch.setenv("PPC_LOCAL_DIRECT", "0")
    monkeypatch.setenv("PPC_STEP_INPLACE", "1")
    n = 3 * (64 << 10) + 1234
    comms, Y, DX = _xor_step(S, M, n, K=K)
    mask = _masks(n)
    Yo, DXo, _, _ = run_1f1b(S, M, K, xor_stage(mask, 0), xor_stage(mask, 1),
                             lambda m: P.source_activation(42, 0, m, n),
                             lambda m: P.source_gradient(42, 0, m, n), n, n, n)
    for m in range(M):
        assert np.array_equal(_host(Y[m])[:n], Yo[m]), m
        assert np.array_equal(_host(DX[m])[:n], DXo[m]), m
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("direct", [1, 0])
@pytest.mark.parametrize("fn", [True, False])
@pytest.mark.parametrize("S", [2, 3])
def test_step_with_host_buffers(S, fn, direct, monkeypatch):
    """The e2e path: pinned HOST inputs X / G and outputs Y / DX.  Host inputs are staged
    into the step buffers, terminal outputs leave on the device->host stream while the next
    ops proceed; repeated steps exercise buffer reuse behind those copies.  fn=True: XOR
    stage functions (outputs via the stage-output buffers); fn=False: identity."""
    monkeypatch.setenv("PPC_LOCAL_DIRECT", str(direct))
    M, n = 6, 2 * (64 << 10) + 777
    cfg = ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=64 << 10)
    comms = ppc.virtual_stages(cfg, DEV)
    hX = [torch.from_numpy(P.source_activation(42, 0, m, n).copy()).pin_memory() for m in range(M)]
    hG = [torch.from_numpy(P.source_gradient(42, 0, m, n).copy()).pin_memory() for m in range(M)]
    hY = [torch.zeros(n, dtype=torch.uint8).pin_memory() for _ in range(M)]
    hDX = [torch.zeros(n, dtype=torch.uint8).pin_memory() for _ in range(M)]
    ctx = [(ppc.XorCtx(42, 0, s, 0), ppc.XorCtx(42, 0, s, 1)) for s in range(S)]
    args = [ppc.StepArgs(M, n, n, fwd=ppc.STAGE_XOR if fn else None,
                         bwd=ppc.STAGE_XOR if fn else None,
                         fwd_user=ctx[s][0] if fn else None, bwd_user=ctx[s][1] if fn else None,
                         x=hX if s == 0 else None, g=hG if s == S - 1 else None,
                         y=hY if s == S - 1 else None, dx=hDX if s == 0 else None)
            for s in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    mask = _masks(n)
    ident = lambda s_, m, x: x
    f = xor_stage(mask, 0) if fn else ident
    b = xor_stage(mask, 1) if fn else ident
    Yo, DXo, _, _ = run_1f1b(S, M, 2, f, b, lambda m: P.source_activation(42, 0, m, n),
                             lambda m: P.source_gradient(42, 0, m, n), n, n, n)
    for _ in range(3):
        for t in hY + hDX:
            t.zero_()
        torch.cuda.synchronize()
        ppc.step_1f1b_local(comms, args, streams)
        torch.cuda.synchronize()
        for m in range(M):
            assert np.array_equal(hY[m].numpy(), Yo[m]), m
            assert np.array_equal(hDX[m].numpy(), DXo[m]), m
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("direct", [1, 0])
@pytest.mark.parametrize("S", [2, 3])
def test_xor_step_cuda_graph(S, direct, monkeypatch):
    """A step captured into a CUDA graph (relative sequence numbers on device) replays
    correctly several times, interleaved with eager steps (host counters stay in sync)."""
    monkeypatch.setenv("PPC_LOCAL_DIRECT", str(direct))
    M, n = 4, 2 * (64 << 10) + 321
    cfg = ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=64 << 10)
    comms = ppc.virtual_stages(cfg, DEV)
    X = [_buf(n) for _ in range(M)]
    G = [_buf(n) for _ in range(M)]
    Y = [_buf(n) for _ in range(M)]
    DX = [_buf(n) for _ in range(M)]
    for m in range(M):
        ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    torch.cuda.synchronize()        # inputs (legacy stream) before the stage streams
    ctx = [(ppc.XorCtx(42, 0, s, 0), ppc.XorCtx(42, 0, s, 1)) for s in range(S)]
    args = [ppc.StepArgs(M, n, n, fwd=ppc.STAGE_XOR, bwd=ppc.STAGE_XOR, fwd_user=ctx[s][0],
                         bwd_user=ctx[s][1], x=X if s == 0 else None, g=G if s == S - 1 else None,
                         y=Y if s == S - 1 else None, dx=DX if s == 0 else None) for s in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    mask = _masks(n)
    ref = [xor_closed_form(S, m, P.source_activation(42, 0, m, n), P.source_gradient(42, 0, m, n),
                           mask) for m in range(M)]

    def check():
        torch.cuda.synchronize()
        for m in range(M):
            assert np.array_equal(_host(Y[m])[:n], ref[m][0]), m
            assert np.array_equal(_host(DX[m])[:n], ref[m][1]), m
            Y[m].fill_(0)
            DX[m].fill_(0)
        torch.cuda.synchronize()

    ppc.step_1f1b_local(comms, args, streams)        # eager step: allocates step buffers
    check()
    g = ppc.StepGraph(comms, args, streams)
    for _ in range(3):
        g.launch()
        check()
    ppc.step_1f1b_local(comms, args, streams)        # eager again after graph launches
    check()
    g.launch()
    check()
    for c in comms:
        assert c.poll() == 0
    g.destroy()
    for c in comms:
        c.disconnect()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("direct", [1, 0])
def test_c2_full_size_sampled(direct, monkeypatch):
    """BASELINE configs[1] shape: [1,4096,4096] bf16 boundary (32 MiB), PP=2, M=8, in the
    launch configuration bench.py times at N=1 (128 KiB chunks, direct single-copy hand-off;
    and the ring path); outputs of micro-batches 0 and 7 compared with the oracle closed
    form byte for byte."""
    monkeypatch.setenv("PPC_LOCAL_DIRECT", str(direct))
    S, M, n = 2, 8, 4096 * 4096 * 2
    comms, Y, DX = _xor_step(S, M, n, chunk=128 << 10)
    mask = _masks(n)
    for m in (0, M - 1):
        y, g = xor_closed_form(S, m, P.source_activation(42, 0, m, n),
                               P.source_gradient(42, 0, m, n), mask)
        assert hashlib.blake2b(_host(Y[m]).tobytes()).digest() == hashlib.blake2b(y.tobytes()).digest()
        assert np.array_equal(_host(DX[m]), g)
    for c in comms:
        c.disconnect()
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("K", [1, 3])
def test_batched_receive_virtual_stages(K):
    """ppc_pp_recv_batch on event-ordered virtual stages (ring path): all n sends enqueued
    first (WOULD_BLOCK otherwise), ragged sizes, bit-exact."""
    sizes = [5, 3 * 65536 + 17, 65536, (1 << 20) + 3]
    comms = _pair(max_msg_bytes=2 << 20, ring_slots=max(K, len(sizes)), chunk_bytes=64 << 10)
    s = torch.cuda.current_stream()
    outs = [_buf(n) for n in sizes]
    assert comms[1].pp_recv(ppc.FWD, outs[0], sizes[0], 0, s) == ppc.WOULD_BLOCK
    srcs = []
    for i, n in enumerate(sizes):
        b = _buf(n)
        srcs.append(b)
        ppc.fill_payload(b, n, 42, 0, 0, 0, i)
        comms[0].send(ppc.FWD, b, n, mb=i, stream=s)
    comms[1].recv_batch(ppc.FWD, outs, sizes, mb0=0, stream=s)
    for i, n in enumerate(sizes):
        assert np.array_equal(_host(outs[i])[:n], P.payload_bytes(42, 0, 0, 0, i, n)), i
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()
