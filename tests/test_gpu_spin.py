"""The cross-process protocol on ONE GPU (cfg.local_spin): every rank of the grid is a comm of
this process, but the comms behave exactly as one process per GPU — device flag / credit /
header spins with .sys scope, zero-copy publication and NVLink-style pulls, TP gathers, the
per-rank step driver (ppc_step_1f1b on each comm, the host never blocks), CUDA graphs per
rank, bounded waits and the sticky error word.  Everything is compared element by element
with the oracle (oracle/transfer.py, oracle/proxy.py, oracle/collectives.py) on the same
seeded inputs (synth/payload.py), bit-exact.  tests/test_gpu_multi.py runs the same protocol
across processes (ranks share the GPU when fewer GPUs than ranks are visible)."""
import hashlib

import time

import numpy as np
import pytest
import torch

import paper_2602_18007_b200 as ppc
from oracle.collectives import allreduce_reference, tp_gather_reference
from oracle.proxy import run_1f1b, xor_closed_form, xor_stage
from synth import payload as P

pytestmark = pytest.mark.gpu

DEV = 0


def _host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint8).reshape(-1)


def _buf(n):
    return torch.empty(max(n, 1), dtype=torch.uint8, device=f"cuda:{DEV}")


def _comms(**kw):
    kw.setdefault("pp", 2)
    cfg = ppc.make_config(local_spin=1, **kw)
    return ppc.local_comms(cfg, DEV)


def _close(comms, expect_ok=True):
    torch.cuda.synchronize()
    if expect_ok:
        for c in comms:
            assert c.poll() == 0, c.error_info()
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


@pytest.mark.parametrize("engine", [ppc.ENGINE_SM, ppc.ENGINE_CE, ppc.ENGINE_PULL])
@pytest.mark.parametrize("K", [1, 2, 3])
def test_send_recv_device_spins(engine, K):
    """Every receive of a direction is enqueued BEFORE its send (on another stream), so each
    one spins on the device until the header / chunk flags land; with K < messages the
    sends wait on device for the receiver's credits.  Ragged sizes, both directions at once,
    every message byte-exact; the trace records show exactly-once in-order delivery."""
    sizes = [0, 1, 100, 65536, 3 * 65536 + 17, (5 << 20) + 3, 4096]
    comms = _comms(max_msg_bytes=8 << 20, ring_slots=K, chunk_bytes=64 << 10, engine=engine,
                   channels=2 if engine == ppc.ENGINE_CE else 1, trace=1)
    st = {(r, k): torch.cuda.Stream() for r in (0, 1) for k in ("send", "recv")}
    outs = {}
    for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
        for i, n in enumerate(sizes):
            outs[(d, i)] = _buf(n)
            outs[(d, i)].fill_(0xAB)
    torch.cuda.synchronize()        # the fills (legacy stream) before the receives
    for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
        for i, n in enumerate(sizes):
            comms[rcv].recv(d, outs[(d, i)], n, mb=i, stream=st[(rcv, "recv")])
    srcs = []
    for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
        for i, n in enumerate(sizes):
            src = _buf(n)
            srcs.append(src)
            ppc.fill_payload(src, n, 42, 0, 0, d, i, stream=st[(snd, "send")])
            comms[snd].send(d, src, n, mb=i, stream=st[(snd, "send")])
    torch.cuda.synchronize()
    for (d, i), t in outs.items():
        n = sizes[i]
        assert np.array_equal(_host(t)[:n], P.payload_bytes(42, 0, 0, d, i, n)), (d, i, n)
    for r, c in enumerate(comms):
        assert c.poll() == 0, c.error_info()
        recs = [x for x in c.trace() if x["kind"] == 1]
        assert [x["seq"] for x in recs] == list(range(1, len(sizes) + 1))
        assert [x["mb"] for x in recs] == list(range(len(sizes)))
        assert all(x["src"] == 1 - r for x in recs)
    _close(comms)


def test_recv_timeout_latches_sticky_error():
    """A receive whose message never comes: the bounded device spin (cfg.timeout_ns) expires,
    PPC_ERR_TIMEOUT latches with the message seq and the wait site (0x100 = header wait);
    every later call on the comm fails with PPC_ERR_STATE (P:L211 hang guard)."""
    comms = _comms(max_msg_bytes=1 << 20, timeout_ns=200_000_000)
    b = _buf(4096)
    comms[1].recv(ppc.FWD, b, 4096, mb=0, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert ppc.STATUS[comms[1].poll()] == "TIMEOUT"
    name, seq, info = comms[1].error_info()
    assert (name, seq, info) == ("TIMEOUT", 1, hex(0x100))
    assert comms[1].pp_recv(ppc.FWD, b, 4096, 1, None) == ppc.STATUS.index("STATE")
    assert comms[0].poll() == 0                       # the sender's comm is unaffected
    _close(comms, expect_ok=False)


def test_send_credit_timeout():
    """K = 1 and nobody receives: the second send's credit wait (device spin in the sender's
    memory) expires and latches TIMEOUT on the sender with the send's direction as info."""
    comms = _comms(max_msg_bytes=1 << 20, ring_slots=1, timeout_ns=200_000_000)
    s = torch.cuda.current_stream()
    b = _buf(4096)
    comms[0].send(ppc.FWD, b, 4096, mb=0, stream=s)
    comms[0].send(ppc.FWD, b, 4096, mb=1, stream=s)
    torch.cuda.synchronize()
    assert comms[0].error_info() == ("TIMEOUT", 2, hex(ppc.FWD))
    _close(comms, expect_ok=False)


def test_header_errors_on_device():
    """SIZE_MISMATCH and ORDER detected by the receive kernel's header check."""
    comms = _comms(max_msg_bytes=1 << 20, timeout_ns=2_000_000_000)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    src, dst = _buf(4096), _buf(4096)
    comms[0].send(ppc.FWD, src, 4096, mb=0, stream=s0)
    comms[1].recv(ppc.FWD, dst, 2048, mb=0, stream=s1)
    torch.cuda.synchronize()
    assert comms[1].error_info()[:2] == ("SIZE_MISMATCH", 1)
    _close(comms, expect_ok=False)
    comms = _comms(max_msg_bytes=1 << 20, timeout_ns=2_000_000_000)
    comms[0].send(ppc.FWD, src, 4096, mb=3, stream=s0)
    comms[1].recv(ppc.FWD, dst, 4096, mb=4, stream=s1)
    torch.cuda.synchronize()
    assert comms[1].error_info()[:2] == ("ORDER", 1)
    _close(comms, expect_ok=False)


def test_latched_error_aborts_queued_waits():
    """One failure poisons the comm and every other bounded wait of it gives up at its next
    check: after a header ORDER error, three more receives queued on the same stream (whose
    messages never come) end within a fraction of their 3 s timeout each, and the latched
    record stays the first failure's."""
    comms = _comms(max_msg_bytes=1 << 20, timeout_ns=3_000_000_000)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    src = _buf(4096)
    dst = [_buf(4096) for _ in range(4)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(4):                     # all queued before anything fails
        comms[1].recv(ppc.FWD, dst[i], 4096, mb=4 + i, stream=s1)
    comms[0].send(ppc.FWD, src, 4096, mb=3, stream=s0)   # mb 3 != 4: ORDER on the first
    torch.cuda.synchronize()
    elapsed = time.perf_counter() - t0
    assert comms[1].error_info()[:2] == ("ORDER", 1)
    assert elapsed < 1.5, elapsed           # not 3 x 3 s of timeouts
    _close(comms, expect_ok=False)


def _xor_args(comms, S, M, n, host_io=False, fn=True):
    X = [_buf(n) for _ in range(M)]
    G = [_buf(n) for _ in range(M)]
    for m in range(M):
        ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    if host_io:
        X = [torch.from_numpy(_host(t)[:n].copy()).pin_memory() for t in X]
        G = [torch.from_numpy(_host(t)[:n].copy()).pin_memory() for t in G]
        Y = [torch.zeros(n, dtype=torch.uint8).pin_memory() for _ in range(M)]
        DX = [torch.zeros(n, dtype=torch.uint8).pin_memory() for _ in range(M)]
    else:
        Y = [_buf(n) for _ in range(M)]
        DX = [_buf(n) for _ in range(M)]
    torch.cuda.synchronize()        # inputs (legacy stream) ready before the stage streams
    ctx = [(ppc.XorCtx(42, 0, s, 0), ppc.XorCtx(42, 0, s, 1)) for s in range(S)]
    args = [ppc.StepArgs(M, n, n, fwd=ppc.STAGE_XOR if fn else None,
                         bwd=ppc.STAGE_XOR if fn else None,
                         fwd_user=ctx[s][0] if fn else None, bwd_user=ctx[s][1] if fn else None,
                         x=X if s == 0 else None, g=G if s == S - 1 else None,
                         y=Y if s == S - 1 else None, dx=DX if s == 0 else None)
            for s in range(S)]
    return args, X, G, Y, DX


def _step_all(comms, args, streams):
    """The per-rank step driver on every stage, enqueued one stage after another."""
    for c, a, s in zip(comms, args, streams):
        ppc.step_1f1b(c, a, s)


def _oracle_xor(S, M, n, K=2, fn=True):
    mask = _masks(n)
    ident = lambda s_, m, x: x
    Yo, DXo, _, _ = run_1f1b(S, M, K, xor_stage(mask, 0) if fn else ident,
                             xor_stage(mask, 1) if fn else ident,
                             lambda m: P.source_activation(42, 0, m, n),
                             lambda m: P.source_gradient(42, 0, m, n), n, n, n)
    return Yo, DXo, mask


@pytest.mark.parametrize("engine", [ppc.ENGINE_SM, ppc.ENGINE_CE, ppc.ENGINE_PULL])
@pytest.mark.parametrize("S,M,K", [(2, 1, 0), (2, 6, 0), (3, 4, 2), (4, 8, 0), (5, 3, 1)])
def test_per_rank_step_driver_xor(engine, S, M, K):
    """ppc_step_1f1b on each stage (the one-process-per-GPU driver) over device spins: XOR
    stage functions, two steps (sequence numbers continue), outputs vs the oracle's 1F1B
    byte simulation and the XOR closed form; receive records exactly once, in order."""
    n = 3 * (64 << 10) + 1234
    comms = _comms(pp=S, max_msg_bytes=n, ring_slots=K, chunk_bytes=64 << 10, engine=engine,
                   channels=2 if engine == ppc.ENGINE_CE else 1, trace=1)
    args, X, G, Y, DX = _xor_args(comms, S, M, n)
    streams = [torch.cuda.Stream() for _ in range(S)]
    Yo, DXo, mask = _oracle_xor(S, M, n, K=K or S + 1)
    for step in range(2):
        _step_all(comms, args, streams)
        torch.cuda.synchronize()
        for m in range(M):
            assert np.array_equal(_host(Y[m])[:n], Yo[m]), (step, m)
            assert np.array_equal(_host(DX[m])[:n], DXo[m]), (step, m)
            y, g = xor_closed_form(S, m, P.source_activation(42, 0, m, n),
                                   P.source_gradient(42, 0, m, n), mask)
            assert np.array_equal(Yo[m], y) and np.array_equal(DXo[m], g)
            Y[m].fill_(0)
            DX[m].fill_(0)
        torch.cuda.synchronize()
    for c in comms:
        assert c.poll() == 0, c.error_info()
        recs = [r for r in c.trace() if r["kind"] == 1]
        for src in (c.rank - 1, c.rank + 1):
            rs = [r for r in recs if r["src"] == src]
            assert [r["seq"] for r in rs] == list(range(1, len(rs) + 1))
            assert [r["mb"] for r in rs] == list(range(M)) * (len(rs) // M)
    _close(comms)


@pytest.mark.parametrize("mode", ["fused", "unfused", "side", "early", "batch", "nochain",
                                  "lastworker", "static"])
def test_zero_copy_publication_and_pull(mode, monkeypatch):
    """Registered send buffers: the sender only publishes (segment, offset) in the receiver's
    slot header, the receiver pulls the payload straight into its buffer.  Ragged messages
    both directions (rendezvous: each send completes when its receive consumed it), then an
    identity 1F1B step whose X / G are registered, two steps.  fused: the step driver
    publishes from the preceding terminal receive kernel (default); unfused: its own
    publication kernel (PPC_FUSE_PUBLISH=0); side: publication on the send stream
    (PPC_ZC_SIDE=1); early: receives look for the publication before griddepcontrol.wait
    (PPC_RECV_EARLY=1); batch: the step's terminal receives with their fused publications
    as one batched-receive grid (PPC_STEP_BATCH=1); the fallbacks of the final per-hop
    changes: nochain (PPC_RECV_CHAIN=0: every receive waits at griddepcontrol.wait),
    lastworker (PPC_PUB_BLOCK0=0: the last worker releases the fused publication behind its
    own system fence), static (PPC_PULL_DYN=0: static chunk ranges per CTA)."""
    env = {"unfused": ("PPC_FUSE_PUBLISH", "0"), "side": ("PPC_ZC_SIDE", "1"),
           "early": ("PPC_RECV_EARLY", "1"), "batch": ("PPC_STEP_BATCH", "1"),
           "nochain": ("PPC_RECV_CHAIN", "0"), "lastworker": ("PPC_PUB_BLOCK0", "0"),
           "static": ("PPC_PULL_DYN", "0")}
    if mode in env:
        monkeypatch.setenv(*env[mode])
    comms = _comms(max_msg_bytes=8 << 20, chunk_bytes=256 << 10, trace=1)
    sizes = [1, 4096 + 3, 3 * (256 << 10) + 5, 8 << 20]
    src = {r: [_buf(n) for n in sizes] for r in (0, 1)}
    for r in (0, 1):
        for i, n in enumerate(sizes):
            ppc.fill_payload(src[r][i], n, 42, 0, 0, r, i)
    torch.cuda.synchronize()
    ppc.register_local(comms, [src[0], src[1]])
    st = [torch.cuda.Stream() for _ in range(4)]
    outs = {}
    for rep in range(2):
        for i, n in enumerate(sizes):
            mb = rep * len(sizes) + i
            for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
                outs[(d, mb)] = _buf(n)
                comms[snd].send(d, src[snd][i], n, mb=mb, stream=st[2 * snd])
                comms[rcv].recv(d, outs[(d, mb)], n, mb=mb, stream=st[2 * rcv + 1])
    torch.cuda.synchronize()
    for (d, mb), t in outs.items():
        i = mb % len(sizes)
        assert np.array_equal(_host(t)[:sizes[i]], P.payload_bytes(42, 0, 0, d, i, sizes[i]))
    M, n = 4, 2 * (256 << 10) + 77
    args, X, G, Y, DX = _xor_args(comms, 2, M, n, fn=False)
    ppc.register_local(comms, [X, G])
    streams = [torch.cuda.Stream() for _ in range(2)]
    for _ in range(2):
        _step_all(comms, args, streams)
        torch.cuda.synchronize()
        for m in range(M):
            assert np.array_equal(_host(Y[m])[:n], P.source_activation(42, 0, m, n)), m
            assert np.array_equal(_host(DX[m])[:n], P.source_gradient(42, 0, m, n)), m
            Y[m].fill_(0)
            DX[m].fill_(0)
        torch.cuda.synchronize()
    # zero-copy receive records start when the publication is seen
    for c in comms:
        assert all(r["t_end_ns"] >= r["t_start_ns"] > 0 for r in c.trace() if r["kind"] == 1)
    _close(comms)


def test_zero_copy_fresh_content_per_message(monkeypatch):
    """a registered source rewritten with NEW content before every message (the
    next write waits until the previous message was consumed, ppc_pp_wait_consumed), with
    the early receive on, so a stale or wrongly applied early pull cannot pass."""
    monkeypatch.setenv("PPC_RECV_EARLY", "1")
    comms = _comms(max_msg_bytes=4 << 20, chunk_bytes=256 << 10, zc_async=1)
    n = (4 << 20) - 13
    src = _buf(n)
    ppc.register_local(comms, [[src], []])
    s_send, s_recv = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for mb in range(6):
        ppc.fill_payload(src, n, 42, 0, 0, 0, mb, stream=s_send)       # new content
        comms[0].send(ppc.FWD, src, n, mb=mb, stream=s_send)
        out = _buf(n)
        outs.append(out)
        comms[1].recv(ppc.FWD, out, n, mb=mb, stream=s_recv)
        comms[0].wait_consumed(ppc.FWD, s_send)                       # before rewriting
    torch.cuda.synchronize()
    for mb, out in enumerate(outs):
        assert np.array_equal(_host(out)[:n], P.payload_bytes(42, 0, 0, 0, mb, n)), mb
    _close(comms)


def test_zero_copy_async_stream():
    """cfg.zc_async: sends complete at publication, a stream of them overlaps; distinct
    registered buffers, both directions at once, every receive enqueued before the sends."""
    sizes = [1, 4096 + 3, 3 * (256 << 10) + 5, 8 << 20, 5 << 20]
    comms = _comms(max_msg_bytes=8 << 20, chunk_bytes=256 << 10, zc_async=1)
    src = {r: [_buf(n) for n in sizes] for r in (0, 1)}
    for r in (0, 1):
        for i, n in enumerate(sizes):
            ppc.fill_payload(src[r][i], n, 42, 0, 0, r, i)
    torch.cuda.synchronize()
    ppc.register_local(comms, [src[0], src[1]])
    st = [torch.cuda.Stream() for _ in range(4)]
    outs = {}
    for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
        for i, n in enumerate(sizes):
            outs[(d, i)] = _buf(n)
            comms[rcv].recv(d, outs[(d, i)], n, mb=i, stream=st[2 * rcv + 1])
    for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
        for i, n in enumerate(sizes):
            comms[snd].send(d, src[snd][i], n, mb=i, stream=st[2 * snd])
        comms[snd].wait_consumed(d, st[2 * snd])
    torch.cuda.synchronize()
    for (d, i), t in outs.items():
        assert np.array_equal(_host(t)[:sizes[i]], P.payload_bytes(42, 0, 0, d, i, sizes[i]))
    _close(comms)


@pytest.mark.parametrize("batch", [0, 1])
@pytest.mark.parametrize("S", [2, 3])
@pytest.mark.parametrize("zc", [False, True])
def test_per_rank_cuda_graph(S, zc, batch, monkeypatch):
    _per_rank_cuda_graph(S, zc, batch, "default", monkeypatch)


@pytest.mark.parametrize("S", [2, 3])
def test_per_rank_cuda_graph_legacy_hops(S, monkeypatch):
    _per_rank_cuda_graph(S, True, 0, "legacy", monkeypatch)


def _per_rank_cuda_graph(S, zc, batch, hop, monkeypatch):
    """Each rank's step captured into its own CUDA graph (ppc_graph_create with n = 1, the
    one-process-per-GPU form; device-side sequence bases), replayed interleaved with eager
    steps.  zc: identity stages with registered X / G (zero-copy pulls and the fused
    publication inside the graphs); otherwise XOR stages over the ring.  batch: terminal
    receives as one batched-receive grid per step (PPC_STEP_BATCH=1).  legacy: without the
    final per-hop changes (no chained receives, last-worker publication, static pull ranges);
    default: with them (chained receives resolve their predecessor's seq on the device)."""
    monkeypatch.setenv("PPC_STEP_BATCH", str(batch))
    if hop == "legacy":
        for k in ("PPC_RECV_CHAIN", "PPC_PUB_BLOCK0", "PPC_PULL_DYN"):
            monkeypatch.setenv(k, "0")
    M, n = 4, 3 * (256 << 10) + 99
    comms = _comms(pp=S, max_msg_bytes=n, chunk_bytes=256 << 10)
    args, X, G, Y, DX = _xor_args(comms, S, M, n, fn=not zc)
    if zc:
        ppc.register_local(comms, [X] + [[]] * (S - 2) + [G])
    streams = [torch.cuda.Stream() for _ in range(S)]
    Yo, DXo, _ = _oracle_xor(S, M, n, K=S + 1, fn=not zc)

    def check():
        torch.cuda.synchronize()
        for c in comms:
            assert c.poll() == 0, c.error_info()
        for m in range(M):
            assert np.array_equal(_host(Y[m])[:n], Yo[m]), m
            assert np.array_equal(_host(DX[m])[:n], DXo[m]), m
            Y[m].fill_(0)
            DX[m].fill_(0)
        torch.cuda.synchronize()

    _step_all(comms, args, streams)              # eager step: allocates the step buffers
    check()
    graphs = [ppc.StepGraph([c], [a], [s]) for c, a, s in zip(comms, args, streams)]
    for it in range(4):
        for g in graphs:
            g.launch()
        check()
        if it == 1:
            _step_all(comms, args, streams)
            check()
    for g in graphs:
        g.destroy()
    _close(comms)


@pytest.mark.parametrize("fn", [True, False])
@pytest.mark.parametrize("S", [2, 3])
def test_per_rank_step_host_buffers(S, fn):
    """The e2e path under the per-rank driver: pinned HOST X / G in, HOST Y / DX out, three
    steps (staging buffers reused behind the host->device / device->host streams); a middle
    stage forwards zero-copy from its step buffers in the arena."""
    M, n = 6, 3 * (64 << 10) + 321
    comms = _comms(pp=S, max_msg_bytes=n, chunk_bytes=64 << 10)
    args, X, G, Y, DX = _xor_args(comms, S, M, n, host_io=True, fn=fn)
    streams = [torch.cuda.Stream() for _ in range(S)]
    Yo, DXo, _ = _oracle_xor(S, M, n, K=S + 1, fn=fn)
    for _ in range(3):
        for t in Y + DX:
            t.zero_()
        torch.cuda.synchronize()
        _step_all(comms, args, streams)
        torch.cuda.synchronize()
        for m in range(M):
            assert np.array_equal(Y[m].numpy(), Yo[m]), m
            assert np.array_equal(DX[m].numpy(), DXo[m]), m
    _close(comms)


@pytest.mark.parametrize("S", [2, 4])
def test_produce_in_place_chain(S):
    """Produce-in-place sends along a chain (the receiver's slot handed to the producer):
    even mb by the fused XOR-send kernel (per-chunk flags from the producer), odd mb by the
    XOR stage writing into the slot + ppc_pp_send_end releasing the flags; every stage on
    its own stream, each receive spinning until its producer's flags land."""
    n, M = 5 * (64 << 10) + 777, 4
    comms = _comms(pp=S, max_msg_bytes=n, chunk_bytes=64 << 10)
    streams = [torch.cuda.Stream() for _ in range(S)]
    mask = _masks(n)
    finals = {}
    keep = []
    import ctypes as C
    xor = ppc._lib.ppc_stage_xor
    xor.restype = C.c_int
    xor.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t,
                    C.c_void_p]
    for m in range(M):
        for d in (ppc.FWD, ppc.BWD):
            order = range(S) if d == ppc.FWD else range(S - 1, -1, -1)
            for k, r in enumerate(order):
                s = streams[r]
                x = _buf(n)
                keep.append(x)
                if k == 0:
                    ppc.fill_payload(x, n, 42, 0, 0, d, m, stream=s)
                else:
                    comms[r].recv(d, x, n, mb=m, stream=s)
                if k == S - 1:
                    finals[(d, m)] = x
                    continue
                ctx = ppc.XorCtx(42, 0, r, d)
                keep.append(ctx)
                if m % 2 == 0:
                    comms[r].xor_send(d, ctx, m, x, n, stream=s)
                else:
                    sl = comms[r].send_begin(d, n, m, stream=s)
                    assert xor(C.byref(ctx), m, x.data_ptr(), sl.payload, n, n, s.cuda_stream) == 0
                    comms[r].send_end(d, False, stream=s)
    torch.cuda.synchronize()
    for (d, m), x in finals.items():
        want = P.payload_bytes(42, 0, 0, d, m, n)
        for st in (range(S - 1) if d == ppc.FWD else range(S - 1, 0, -1)):
            want = want ^ mask(st, d, m)
        assert np.array_equal(_host(x)[:n], want), (d, m)
    _close(comms)


def test_step_produce_in_place(monkeypatch):
    """PPC_STEP_INPLACE=1 under the per-rank driver: stage fns write into the receiver's slot."""
    monkeypatch.setenv("PPC_STEP_INPLACE", "1")
    S, M, n = 3, 6, 5 * (64 << 10) + 777
    comms = _comms(pp=S, max_msg_bytes=n, chunk_bytes=64 << 10)
    args, X, G, Y, DX = _xor_args(comms, S, M, n)
    streams = [torch.cuda.Stream() for _ in range(S)]
    Yo, DXo, _ = _oracle_xor(S, M, n, K=S + 1)
    _step_all(comms, args, streams)
    torch.cuda.synchronize()
    for m in range(M):
        assert np.array_equal(_host(Y[m])[:n], Yo[m]), m
        assert np.array_equal(_host(DX[m])[:n], DXo[m]), m
    _close(comms)


def test_tp_sliced_gather():
    """NEXT-1, PP=2 x TP=2 as four comms on one GPU: each TP rank sends only its half of the
    boundary (zero-copy), each TP rank of the other stage gathers both halves (pulled, fused
    all-gather); compared with the oracle's definition (concatenation of the TP slices),
    both directions, ragged slices, several messages."""
    tp = 2
    comms = _comms(tp=tp, pp=2, max_msg_bytes=4 << 20, chunk_bytes=256 << 10)
    slice_n = 3 * (256 << 10) + 77
    total = tp * slice_n
    M = 3
    fulls, outs = {}, {}
    for r, c in enumerate(comms):
        pp_i = r // tp
        d_send = ppc.FWD if pp_i == 0 else ppc.BWD
        fulls[r] = [_buf(total) for _ in range(M)]
        for m in range(M):
            ppc.fill_payload(fulls[r][m], total, 42, 0, P.SRC_BOUNDARY, d_send, m)
    torch.cuda.synchronize()
    ppc.register_local(comms, [fulls[r] for r in range(len(comms))])
    st = {(r, k): torch.cuda.Stream() for r in range(len(comms)) for k in (0, 1)}
    for m in range(M):
        for r, c in enumerate(comms):
            pp_i, tp_i = r // tp, r % tp
            d_send = ppc.FWD if pp_i == 0 else ppc.BWD
            d_recv = 1 - d_send
            c.send(d_send, fulls[r][m].data_ptr() + tp_i * slice_n, slice_n, mb=m,
                   stream=st[(r, 0)])
            outs[(r, m)] = _buf(total)
            c.recv_gather(d_recv, outs[(r, m)], total, mb=m, stream=st[(r, 1)])
    torch.cuda.synchronize()
    for (r, m), out in outs.items():
        d_recv = ppc.BWD if r // tp == 0 else ppc.FWD
        full = P.payload_bytes(42, 0, P.SRC_BOUNDARY, d_recv, m, total)
        ref = tp_gather_reference([full[t * slice_n:(t + 1) * slice_n] for t in range(tp)])
        assert np.array_equal(_host(out), ref), (r, m)
    _close(comms)


@pytest.mark.parametrize("S", [2, 3])
def test_hetero_allreduce_leader_chain(S):
    """NEXT-2 with DP = 1: the cross-subgroup exchange over the PP peer path (reduce forward
    along the stage chain, result backward); exact against the oracle's plain sum in
    ascending-rank order (integer-valued fp32, and int32)."""
    comms = _comms(pp=S, max_msg_bytes=8 << 20)
    n = (1 << 20) + 3
    idx = np.arange(n, dtype=np.int64)
    vals = {r: ((r + 1) * (idx % 7 + 1)).astype(np.float32) for r in range(S)}
    ref = allreduce_reference(vals, list(range(S)))
    streams = [torch.cuda.Stream() for _ in range(S)]
    for dtype, tdt in ((7, torch.float32), (2, torch.int32)):
        ts = [torch.from_numpy(vals[r]).to(tdt).cuda(DEV) for r in range(S)]
        for c, t, s in zip(comms, ts, streams):
            c.hetero_allreduce(t, dtype, stream=s)
        torch.cuda.synchronize()
        for r, t in enumerate(ts):
            assert np.array_equal(t.cpu().numpy().astype(np.float64), ref), (r, dtype)
    _close(comms)


@pytest.mark.parametrize("batch", [0, 1])
def test_full_size_c2_zero_copy_graph(batch, monkeypatch):
    """BASELINE configs[1] at full size in bench.py's N >= 2 launch configuration, run on one
    GPU: [1,4096,4096] bf16 (32 MiB) messages, PP = 2, M = 8, registered X / G (zero-copy
    pulls, 256 KiB grain, fused publication), each rank's step replayed as a CUDA graph.
    ALL 8 Y and 8 DX compared with the oracle byte for byte (blake2b of the full buffers
    plus first / last 4 KiB), over three replays.  batch: PPC_STEP_BATCH=1."""
    monkeypatch.setenv("PPC_STEP_BATCH", str(batch))
    S, M, n = 2, 8, 4096 * 4096 * 2
    comms = _comms(pp=S, max_msg_bytes=n, chunk_bytes=256 << 10)
    args, X, G, Y, DX = _xor_args(comms, S, M, n, fn=False)
    ppc.register_local(comms, [X, G])
    streams = [torch.cuda.Stream() for _ in range(S)]
    ref_y = [P.source_activation(42, 0, m, n) for m in range(M)]
    ref_dx = [P.source_gradient(42, 0, m, n) for m in range(M)]
    dig = lambda a: hashlib.blake2b(a.tobytes(), digest_size=16).digest()
    ref_y_d = [dig(a) for a in ref_y]
    ref_dx_d = [dig(a) for a in ref_dx]
    _step_all(comms, args, streams)
    torch.cuda.synchronize()
    graphs = [ppc.StepGraph([c], [a], [s]) for c, a, s in zip(comms, args, streams)]
    for _ in range(3):
        for g in graphs:
            g.launch()
        torch.cuda.synchronize()
        for c in comms:
            assert c.poll() == 0, c.error_info()
        for m in range(M):
            y, dx = _host(Y[m]), _host(DX[m])
            assert dig(y) == ref_y_d[m] and np.array_equal(y[:4096], ref_y[m][:4096]), m
            assert dig(dx) == ref_dx_d[m] and np.array_equal(dx[-4096:], ref_dx[m][-4096:]), m
            Y[m].fill_(0)
            DX[m].fill_(0)
        torch.cuda.synchronize()
    for g in graphs:
        g.destroy()
    _close(comms)


@pytest.mark.parametrize("zc", [False, True])
@pytest.mark.parametrize("K", [2, 3])
def test_batched_receive(zc, K):
    """ppc_pp_recv_batch: one grid receives n consecutive messages (ragged sizes, n > K so the
    ring wraps inside one batch and the sender waits for the batch's own credits), both
    directions at once; zc: registered sources (zc_async: the sender publishes ahead), else
    SM push into the ring.  Every message byte-exact and recorded once, in order."""
    sizes = [4096 + 3, 3 * (256 << 10) + 5, 1, (2 << 20) + 17, 256 << 10, 5, 777777, 64 << 10]
    comms = _comms(max_msg_bytes=4 << 20, chunk_bytes=256 << 10, ring_slots=K,
                   zc_async=1 if zc else 0, trace=1)
    src = {r: [_buf(n) for n in sizes] for r in (0, 1)}
    for r in (0, 1):
        for i, n in enumerate(sizes):
            ppc.fill_payload(src[r][i], n, 42, 0, 0, r, i)
    torch.cuda.synchronize()
    if zc:
        ppc.register_local(comms, [src[0], src[1]])
    st = [torch.cuda.Stream() for _ in range(4)]
    outs = {}
    for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
        outs[d] = [_buf(n) for n in sizes]
        comms[rcv].recv_batch(d, outs[d][:5], sizes[:5], mb0=0, stream=st[2 * rcv + 1])
        comms[rcv].recv_batch(d, outs[d][5:], sizes[5:], mb0=5, stream=st[2 * rcv + 1])
    for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
        for i, n in enumerate(sizes):
            comms[snd].send(d, src[snd][i], n, mb=i, stream=st[2 * snd])
        comms[snd].wait_consumed(d, st[2 * snd])
    torch.cuda.synchronize()
    for d in (ppc.FWD, ppc.BWD):
        for i, n in enumerate(sizes):
            assert np.array_equal(_host(outs[d][i])[:n], P.payload_bytes(42, 0, 0, d, i, n)), (d, i)
    for r, c in enumerate(comms):
        assert c.poll() == 0, c.error_info()
        recs = [x for x in c.trace() if x["kind"] == 1]
        assert [x["seq"] for x in recs] == list(range(1, len(sizes) + 1))
        assert [x["mb"] for x in recs] == list(range(len(sizes)))
    _close(comms)


def test_batched_receive_header_error():
    """A wrong size inside a batch latches SIZE_MISMATCH with that message's seq."""
    comms = _comms(max_msg_bytes=1 << 20, timeout_ns=2_000_000_000)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    src = _buf(8192)
    outs = [_buf(8192) for _ in range(3)]
    for i in range(3):
        comms[0].send(ppc.FWD, src, 8192, mb=i, stream=s0)
    comms[1].recv_batch(ppc.FWD, outs, [8192, 8192, 4096], mb0=0, stream=s1)
    torch.cuda.synchronize()
    assert comms[1].error_info()[:2] == ("SIZE_MISMATCH", 3)
    _close(comms, expect_ok=False)


def test_early_receive_hits_and_stays_exact(monkeypatch):
    """PPC_RECV_EARLY=1: three zero-copy messages from distinct registered buffers
    are published BEFORE their receives are enqueued back to back on one stream, so the
    receives after the first find their publication in the early look (record dir = -2) and
    pull their first 64 KiB per CTA before griddepcontrol.wait; bytes exact either way."""
    monkeypatch.setenv("PPC_RECV_EARLY", "1")
    n = 4 << 20
    comms = _comms(max_msg_bytes=n, chunk_bytes=256 << 10, zc_async=1, trace=1)
    srcs = [_buf(n) for _ in range(3)]
    for i, b in enumerate(srcs):
        ppc.fill_payload(b, n, 42, 0, 0, 0, i)
    torch.cuda.synchronize()
    ppc.register_local(comms, [srcs, []])
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    for i in range(3):
        comms[0].send(ppc.FWD, srcs[i], n, mb=i, stream=s0)
    torch.cuda.synchronize()                    # all three published
    outs = [_buf(n) for _ in range(3)]
    for i in range(3):
        comms[1].recv(ppc.FWD, outs[i], n, mb=i, stream=s1)
    comms[0].wait_consumed(ppc.FWD, s0)
    torch.cuda.synchronize()
    for i in range(3):
        assert np.array_equal(_host(outs[i]), P.payload_bytes(42, 0, 0, 0, i, n)), i
    recs = [r for r in comms[1].trace() if r["kind"] == 1]
    assert [r["seq"] for r in recs] == [1, 2, 3]
    assert sum(r["dir"] == -2 for r in recs) >= 1, recs
    _close(comms)


@pytest.mark.parametrize("C", [2, 3, 8])
@pytest.mark.parametrize("mode", ["sm", "pull", "zc"])
def test_mpdt_channels(C, mode):
    """MPDT analogue: a message's chunks split into C contiguous channel ranges, each
    moved by its own CTA group (push, PULL staging + pulls, zero-copy pulls); ragged sizes
    with fewer chunks than channels, both directions, byte-exact."""
    engine = {"sm": ppc.ENGINE_SM, "pull": ppc.ENGINE_PULL, "zc": ppc.ENGINE_SM}[mode]
    sizes = [1, 3 * 65536 + 17, (2 << 20) + 5, 65536 * 7]
    comms = _comms(max_msg_bytes=4 << 20, chunk_bytes=64 << 10, engine=engine, channels=C,
                   cta_per_channel=2)
    src = {r: [_buf(n) for n in sizes] for r in (0, 1)}
    for r in (0, 1):
        for i, n in enumerate(sizes):
            ppc.fill_payload(src[r][i], n, 42, 0, 0, r, i)
    torch.cuda.synchronize()
    if mode == "zc":
        ppc.register_local(comms, [src[0], src[1]])
    st = [torch.cuda.Stream() for _ in range(4)]
    outs = {}
    for d, (snd, rcv) in ((ppc.FWD, (0, 1)), (ppc.BWD, (1, 0))):
        for i, n in enumerate(sizes):
            outs[(d, i)] = _buf(n)
            comms[snd].send(d, src[snd][i], n, mb=i, stream=st[2 * snd])
            comms[rcv].recv(d, outs[(d, i)], n, mb=i, stream=st[2 * rcv + 1])
    torch.cuda.synchronize()
    for (d, i), t in outs.items():
        assert np.array_equal(_host(t)[:sizes[i]], P.payload_bytes(42, 0, 0, d, i, sizes[i])), (d, i)
    _close(comms)


@pytest.mark.parametrize("name", ["C4", "C3"])
def test_full_size_north_star_configs_on_one_gpu(name):
    """BASELINE configs[3] C4 (Qwen2-7B [1,4096,3584] bf16, PP = 8, M = 32) and configs[2] C3
    (LLaMA-8B [1,4096,4096], PP = 4 x TP = 2: two TP pipelines, M = 16) at full size with
    bench.py's launch configuration for them (ring push, 512 KiB chunks, K = pp + 1) — every
    rank a comm of this process on one GPU
    under the cross-process protocol.  Identity stages: every Y_m of the last stages equals
    the stage-0 input X_m and every DX_m of stage 0 equals G_m, checked for ALL micro-batches
    against the synth payloads by digest (plus first / last bytes)."""
    import bench
    a = bench.parse([])
    wl = bench.resolve(a, 8, name)
    S, TP, M, n = wl["pp"], wl["tp"], wl["M"], wl["msg_bytes"]
    comms = _comms(tp=TP, pp=S, max_msg_bytes=n, chunk_bytes=wl["chunk"], ring_slots=wl["slots"])
    world = len(comms)
    dig = lambda x: hashlib.blake2b(x.tobytes(), digest_size=16).digest()
    ref_x = [P.source_activation(42, 0, m, n) for m in range(M)]
    ref_g = [P.source_gradient(42, 0, m, n) for m in range(M)]
    dx, dg = [dig(x) for x in ref_x], [dig(g) for g in ref_g]
    X = [_buf(n) for _ in range(M)]
    G = [_buf(n) for _ in range(M)]
    for m in range(M):
        ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    outs = {}
    args = []
    for r, c in enumerate(comms):
        st = c.group(ppc.GROUP_PP)[0].index(r)
        y = [_buf(n) for _ in range(M)] if st == S - 1 else None
        d = [_buf(n) for _ in range(M)] if st == 0 else None
        outs[r] = (y, d)
        args.append(ppc.StepArgs(M, n, n, x=X if st == 0 else None, g=G if st == S - 1 else None,
                                 y=y, dx=d))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(world)]
    # eager steps (8 ranks' graphs would add 8 capture streams: this process must stay under
    # the GPU's 32 hardware queues); the second step runs on allocated buffers
    # with continuing sequence numbers
    for _ in range(2):
        _step_all(comms, args, streams)
        torch.cuda.synchronize()
    for c in comms:
        assert c.poll() == 0, c.error_info()
    checked = 0
    for r, (y, d) in outs.items():
        for bufs, want, ref in ((y, dx, ref_x), (d, dg, ref_g)):
            if bufs is None:
                continue
            for m in range(M):
                h = _host(bufs[m])
                assert dig(h) == want[m] and np.array_equal(h[:4096], ref[m][:4096]), (r, m)
                checked += 1
    assert checked == 2 * TP * M
    _close(comms)
