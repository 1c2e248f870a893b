"""Worker for the multi-GPU parity tests (one process per GPU, launched by torchrun from
tests/test_gpu_multi.py).  Bootstrap over gloo (the host control plane), data over the
libppc peer kernels; each rank checks its own outputs against the oracle and exits
non-zero on any mismatch."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_18007_b200 as ppc  # noqa: E402
from oracle.proxy import xor_closed_form  # noqa: E402
from synth import payload as P  # noqa: E402


def dev(rank):
    """CUDA device of a rank: its own GPU, or (fewer GPUs than ranks, e.g. the 1-GPU driver
    box) GPUs shared round-robin — ranks on one GPU are separate processes, so CUDA IPC,
    device spins and the per-rank step driver run exactly as across GPUs (time-sliced)."""
    return rank % torch.cuda.device_count()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint8).reshape(-1)


def buf(n):
    return torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")


def case_sendrecv(rank, world, engine):
    cfg = ppc.make_config(pp=world, max_msg_bytes=8 << 20, chunk_bytes=256 << 10, engine=engine,
                          channels=4 if engine else 1)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    s = torch.cuda.current_stream()
    sizes = [0, 1, 4096, 3 * (256 << 10) + 5, 8 << 20]
    for rep in range(3):
        for i, n in enumerate(sizes):
            mb = rep * len(sizes) + i
            for d in (ppc.FWD, ppc.BWD):
                sender = rank == 0 if d == ppc.FWD else rank == 1
                receiver = rank == 1 if d == ppc.FWD else rank == 0
                if sender:
                    b = buf(n)
                    ppc.fill_payload(b, n, 42, 0, 0, d, mb)
                    comm.send(d, b, n, mb=mb, stream=s)
                    torch.cuda.synchronize()
                elif receiver:
                    b = buf(n)
                    comm.recv(d, b, n, mb=mb, stream=s)
                    got = host(b)[:n]
                    want = P.payload_bytes(42, 0, 0, d, mb, n)
                    assert np.array_equal(got, want), (rank, d, n, mb)
    torch.cuda.synchronize()
    assert comm.poll() == 0
    return comm


def case_xor(rank, world, engine, M=6):
    S = world
    n = 5 * (256 << 10) + 777
    cfg = ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=256 << 10, engine=engine,
                          channels=2 if engine else 1, trace=1)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    X = [buf(n) for _ in range(M)] if rank == 0 else None
    G = [buf(n) for _ in range(M)] if rank == S - 1 else None
    out = [buf(n) for _ in range(M)]
    for m in range(M):
        if X:
            ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        if G:
            ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    fctx, bctx = ppc.XorCtx(42, 0, rank, 0), ppc.XorCtx(42, 0, rank, 1)
    args = ppc.StepArgs(M, n, n, fwd=ppc.STAGE_XOR, bwd=ppc.STAGE_XOR, fwd_user=fctx,
                        bwd_user=bctx, x=X, g=G, y=out if rank == S - 1 else None,
                        dx=out if rank == 0 else None)
    for step in range(2):                      # two steps: seq numbers continue across steps
        ppc.step_1f1b(comm, args, torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert comm.poll() == 0, ppc.STATUS[comm.poll()]
        if rank in (0, S - 1):
            mask = lambda s, d, m: P.proxy_mask(42, 0, s, d, m, n)
            for m in range(M):
                y, g = xor_closed_form(S, m, P.source_activation(42, 0, m, n),
                                       P.source_gradient(42, 0, m, n), mask)
                want = y if rank == S - 1 else g
                assert np.array_equal(host(out[m])[:n], want), (rank, step, m)
    recs = [r for r in comm.trace() if r["kind"] == 1]
    for src in (rank - 1, rank + 1):
        rs = [r for r in recs if r["src"] == src]
        assert [r["seq"] for r in rs] == list(range(1, len(rs) + 1))
        assert [r["mb"] for r in rs] == list(range(M)) * (len(rs) // M)
    return comm


def case_host(rank, world, M=6):
    """The e2e path across processes: pinned HOST X / G in, HOST Y / DX out, XOR stage
    functions and identity, 3 steps each (staging buffers reused behind the host->device
    and device->host streams); middle stages (world > 2) forward zero-copy from the step
    buffers in their arena."""
    S = world
    n = 3 * (256 << 10) + 321
    cfg = ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=256 << 10)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    pin = lambda a: torch.from_numpy(a.copy()).pin_memory()
    hX = [pin(P.source_activation(42, 0, m, n)) for m in range(M)] if rank == 0 else None
    hG = [pin(P.source_gradient(42, 0, m, n)) for m in range(M)] if rank == S - 1 else None
    hout = [torch.zeros(n, dtype=torch.uint8).pin_memory() for _ in range(M)]
    fctx, bctx = ppc.XorCtx(42, 0, rank, 0), ppc.XorCtx(42, 0, rank, 1)
    mask = lambda s, d, m: P.proxy_mask(42, 0, s, d, m, n)
    for fn in (True, False):
        args = ppc.StepArgs(M, n, n, fwd=ppc.STAGE_XOR if fn else None,
                            bwd=ppc.STAGE_XOR if fn else None,
                            fwd_user=fctx if fn else None, bwd_user=bctx if fn else None,
                            x=hX, g=hG, y=hout if rank == S - 1 else None,
                            dx=hout if rank == 0 else None)
        for step in range(3):
            for t in hout:
                t.zero_()
            ppc.step_1f1b(comm, args, torch.cuda.current_stream())
            torch.cuda.synchronize()
            assert comm.poll() == 0, comm.error_info()
            if rank in (0, S - 1):
                for m in range(M):
                    xs, gs = P.source_activation(42, 0, m, n), P.source_gradient(42, 0, m, n)
                    if fn:
                        y, g = xor_closed_form(S, m, xs, gs, mask)
                    else:
                        y, g = xs, gs
                    want = y if rank == S - 1 else g
                    assert np.array_equal(hout[m].numpy(), want), (rank, fn, step, m)
            dist.barrier()
    return comm


def case_timeout(rank, world):
    cfg = ppc.make_config(pp=world, max_msg_bytes=1 << 20, timeout_ns=300_000_000)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    if rank == 1:
        b = buf(4096)
        comm.recv(ppc.FWD, b, 4096, mb=0, stream=torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert ppc.STATUS[comm.poll()] == "TIMEOUT", comm.poll()
    return comm


def case_dcbs1(rank, world):
    """DCBS with one-rank TP / DP groups, ranks sharing a GPU (the driver's one-GPU box):
    under PPC_NCCL_SINGLETON=1 every group still gets its own NCCL communicator, so the id
    exchange, ncclCommInitRank and ncclAllReduce run through the C ABI beside the PP kernels
    of a 1F1B step; the allreduce over a one-rank group is the identity."""
    assert os.environ.get("PPC_NCCL_SINGLETON") == "1"
    cfg = ppc.make_config(tp=1, pp=world, dp=1, max_msg_bytes=2 << 20)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=True)
    tp_m, be = comm.group(ppc.GROUP_TP)
    dp_m, be_dp = comm.group(ppc.GROUP_DP)
    pp_m, be_pp = comm.group(ppc.GROUP_PP)
    assert tp_m == [rank] and dp_m == [rank] and pp_m == list(range(world))
    assert be == be_dp == ppc.BACKEND_NCCL and be_pp == ppc.BACKEND_PEER
    side = torch.cuda.Stream()
    t = torch.full((1 << 20,), float(rank + 1), device="cuda")
    with torch.cuda.stream(side):
        comm.allreduce(ppc.GROUP_TP, t, 7, stream=side)        # ncclFloat32 = 7
        comm.allreduce(ppc.GROUP_DP, t, 7, stream=side)
    try:
        comm.allreduce(ppc.GROUP_PP, t, 7)
        raise AssertionError("PP allreduce must be refused (DCBS)")
    except ppc.PpcError as e:
        assert e.name == "BACKEND"
    n, M = (1 << 20) + 3, 4
    X = [buf(n) for _ in range(M)] if rank == 0 else None
    G = [buf(n) for _ in range(M)] if rank == world - 1 else None
    for m in range(M):
        if X:
            ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        if G:
            ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    torch.cuda.synchronize()
    out = [buf(n) for _ in range(M)]
    args = ppc.StepArgs(M, n, n, x=X, g=G, y=out if G else None, dx=out if X else None)
    ppc.step_1f1b(comm, args, torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert comm.poll() == 0
    assert torch.all(t == float(rank + 1)).item()
    for m in range(M):      # identity stages: stage 0 gets G_m back, last stage gets X_m
        if X or G:
            ref = P.source_gradient(42, 0, m, n) if X else P.source_activation(42, 0, m, n)
            assert np.array_equal(host(out[m])[:n], ref)
    return comm


def case_dcbs(rank, world):
    """PP=2 x TP=2 on 4 GPUs: TP allreduce on NCCL running beside the PP kernels."""
    tp = 2
    cfg = ppc.make_config(tp=tp, pp=world // tp, dp=1, max_msg_bytes=1 << 20)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=True)
    tp_m, be = comm.group(ppc.GROUP_TP)
    pp_m, be2 = comm.group(ppc.GROUP_PP)
    assert be == ppc.BACKEND_NCCL and be2 == ppc.BACKEND_PEER and len(tp_m) == tp
    with_err = comm
    side = torch.cuda.Stream()
    t = torch.full((1 << 20,), float(rank + 1), device="cuda")
    with torch.cuda.stream(side):
        comm.allreduce(ppc.GROUP_TP, t, 7, stream=side)        # ncclFloat32 = 7
    try:
        comm.allreduce(ppc.GROUP_PP, t, 7)
        raise AssertionError("PP allreduce must be refused (DCBS)")
    except ppc.PpcError as e:
        assert e.name == "BACKEND"
    n = 1 << 20
    M = 4
    pp_rank = pp_m.index(rank)
    X = [buf(n) for _ in range(M)] if pp_rank == 0 else None
    G = [buf(n) for _ in range(M)] if pp_rank == len(pp_m) - 1 else None
    for m in range(M):
        if X:
            ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        if G:
            ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    out = [buf(n) for _ in range(M)]
    args = ppc.StepArgs(M, n, n, x=X, g=G, y=out if G else None, dx=out if X else None)
    ppc.step_1f1b(comm, args, torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert with_err.poll() == 0
    want = sum(range(1, tp + 1)) + tp * tp_m[0]
    assert torch.all(t == float(want)).item(), (t[0].item(), want)
    for m in range(M):      # identity stages: stage 0 gets G_m back, last stage gets X_m
        ref = P.source_gradient(42, 0, m, n) if X else P.source_activation(42, 0, m, n)
        assert np.array_equal(host(out[m])[:n], ref)
    return comm


def case_toy(rank, world, bf16=True, steps=5):
    """C1 toy pipeline across two processes / GPUs; loss vs the oracle (BJ gate 1e-3)."""
    from paper_2602_18007_b200.toy import ToyStage
    from oracle import toy as otoy
    from synth.toy import ROWS, WIDTH, data, init_params
    M = 4
    Ws, bs = init_params(42)
    X, T = data(M, 42)
    st = ToyStage(rank, ROWS, WIDTH, M, 10.0, bf16, dev(rank), Ws[2 * rank:2 * rank + 2],
                  bs[2 * rank:2 * rank + 2], X if rank == 0 else T)
    cfg = ppc.make_config(pp=2, max_msg_bytes=st.boundary_bytes, chunk_bytes=64 << 10)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    s = torch.cuda.current_stream()
    args = st.step_args()
    losses = []
    for _ in range(steps):
        ppc.step_1f1b(comm, args, s)
        if rank == 1:
            losses.append(st.loss(s))
        st.step_end(s)
    torch.cuda.synchronize()
    assert comm.poll() == 0
    if rank == 1:
        ref, _, _ = otoy.train(Ws, bs, X, T, steps, lr=10.0, dtype=np.float64, bf16=bf16)
        rel = max(abs(g - r) / abs(r) for g, r in zip(losses, ref))
        assert rel <= 1e-3, (losses, ref)
        print(f"toy losses {losses} oracle {ref} max rel {rel:.2e}", flush=True)
    st.destroy()
    return comm


def case_zc(rank, world):
    """Zero-copy pulls from registered send buffers: ragged sizes byte-exact, then an identity
    1F1B step whose X / G sources are registered (the receiver pulls them over NVLink)."""
    cfg = ppc.make_config(pp=world, max_msg_bytes=8 << 20, chunk_bytes=256 << 10)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    s = torch.cuda.current_stream()
    sizes = [1, 4096 + 3, 3 * (256 << 10) + 5, 8 << 20]
    src = [buf(n) for n in sizes]
    for i, (b, n) in enumerate(zip(src, sizes)):
        ppc.fill_payload(b, n, 42, 0, 0, rank, i)
    ppc.register_tensors(comm, src)
    for rep in range(3):
        for i, n in enumerate(sizes):
            mb = rep * len(sizes) + i
            for d in (ppc.FWD, ppc.BWD):
                if (d == ppc.FWD and rank == 0) or (d == ppc.BWD and rank == 1):
                    comm.send(d, src[i], n, mb=mb, stream=s)
                elif (d == ppc.FWD and rank == 1) or (d == ppc.BWD and rank == 0):
                    out = buf(n)
                    comm.recv(d, out, n, mb=mb, stream=s)
                    want = P.payload_bytes(42, 0, 0, 1 - rank, i, n)
                    assert np.array_equal(host(out)[:n], want), (rank, d, n, mb)
    torch.cuda.synchronize()
    assert comm.poll() == 0
    M, n = 4, 2 * (256 << 10) + 77
    X = [buf(n) for _ in range(M)] if rank == 0 else None
    G = [buf(n) for _ in range(M)] if rank == 1 else None
    for m in range(M):
        if X:
            ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        if G:
            ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    ppc.register_tensors(comm, X or G)
    out = [buf(n) for _ in range(M)]
    args = ppc.StepArgs(M, n, n, x=X, g=G, y=out if rank == 1 else None, dx=out if rank == 0 else None)
    for _ in range(2):
        ppc.step_1f1b(comm, args, s)
    torch.cuda.synchronize()
    assert comm.poll() == 0
    for m in range(M):
        ref = P.source_gradient(42, 0, m, n) if rank == 0 else P.source_activation(42, 0, m, n)
        assert np.array_equal(host(out[m])[:n], ref), (rank, m)
    return comm


def case_zc_bidir_stream(rank, world):
    """Both directions at once, a stream of zero-copy messages per direction, every receive
    of a direction enqueued before its sends (bench_sweep's bidir mode), with 128- and
    256-CTA receive grids requested.  Regression for a stall until the timeout when the
    spinning receive CTAs in flight exceeded the SM count and the peer's publication kernels
    could no longer be scheduled (libppc now caps cross-GPU receive grids at 64 CTAs,
    profiles/r47_zc_bidir.log)."""
    n, N = 32 << 20, 8
    cfg = ppc.make_config(pp=world, max_msg_bytes=n, chunk_bytes=128 << 10,
                          timeout_ns=5_000_000_000)      # 256 chunks: grids up to 256 CTAs
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    src = buf(n)
    ppc.fill_payload(src, n, 42, 0, 0, rank, 0)
    ppc.register_tensors(comm, [src])
    dst = buf(n)
    s_send, s_recv = torch.cuda.Stream(), torch.cuda.Stream()
    d_out = ppc.FWD if rank == 0 else ppc.BWD
    d_in = ppc.BWD if rank == 0 else ppc.FWD
    for rep in range(4):
        # 128 CTAs: two receive grids fit (PDL on); 256: they do not (PDL off for them)
        os.environ["PPC_RECV_CTAS"] = "128" if rep < 2 else "256"
        torch.cuda.synchronize()
        dist.barrier()
        for i in range(N):
            comm.recv(d_in, dst, n, mb=rep * N + i, stream=s_recv)
        for i in range(N):
            comm.send(d_out, src, n, mb=rep * N + i, stream=s_send)
        torch.cuda.synchronize()
        assert comm.poll() == 0, comm.error_info()
    want = P.payload_bytes(42, 0, 0, 1 - rank, 0, n)
    assert np.array_equal(host(dst)[:n], want)
    os.environ.pop("PPC_RECV_CTAS")
    return comm


def case_zc_async(rank, world):
    """cfg.zc_async: zero-copy sends complete at publication, so a stream of sends overlaps;
    ppc_pp_wait_consumed marks buffer reuse.  Distinct registered buffers per message, both
    directions at once, ragged sizes; every message byte-exact and in order."""
    sizes = [1, 4096 + 3, 3 * (256 << 10) + 5, 8 << 20, 5 << 20]
    cfg = ppc.make_config(pp=world, max_msg_bytes=8 << 20, chunk_bytes=256 << 10, zc_async=1)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    src = [buf(n) for n in sizes]
    for i, (b, n) in enumerate(zip(src, sizes)):
        ppc.fill_payload(b, n, 42, 0, 0, rank, i)
    ppc.register_tensors(comm, src)
    outs = [buf(n) for n in sizes]
    s_send, s_recv = torch.cuda.Stream(), torch.cuda.Stream()
    d_out = ppc.FWD if rank == 0 else ppc.BWD
    d_in = ppc.BWD if rank == 0 else ppc.FWD
    for rep in range(2):
        for i, n in enumerate(sizes):
            comm.recv(d_in, outs[i], n, mb=rep * len(sizes) + i, stream=s_recv)
        for i, n in enumerate(sizes):
            comm.send(d_out, src[i], n, mb=rep * len(sizes) + i, stream=s_send)
        comm.wait_consumed(d_out, s_send)
        torch.cuda.synchronize()
        assert comm.poll() == 0, comm.error_info()
        for i, n in enumerate(sizes):
            assert np.array_equal(host(outs[i])[:n], P.payload_bytes(42, 0, 0, 1 - rank, i, n)), i
            outs[i].zero_()
        torch.cuda.synchronize()
        dist.barrier()
    return comm


def case_graph(rank, world, zc=False):
    """A 1F1B step captured into a CUDA graph across processes (device-side sequence bases):
    XOR step graph launches interleaved with eager steps; then an identity step whose X / G
    are registered (zero-copy pulls inside the graph)."""
    S, M, n = world, 4, 3 * (256 << 10) + 99
    cfg = ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=256 << 10)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    s = torch.cuda.current_stream()
    X = [buf(n) for _ in range(M)] if rank == 0 else None
    G = [buf(n) for _ in range(M)] if rank == S - 1 else None
    out = [buf(n) for _ in range(M)]
    for m in range(M):
        if X:
            ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        if G:
            ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    fctx, bctx = ppc.XorCtx(42, 0, rank, 0), ppc.XorCtx(42, 0, rank, 1)
    xargs = ppc.StepArgs(M, n, n, fwd=ppc.STAGE_XOR, bwd=ppc.STAGE_XOR, fwd_user=fctx,
                         bwd_user=bctx, x=X, g=G, y=out if rank == S - 1 else None,
                         dx=out if rank == 0 else None)
    mask = lambda st, d, m: P.proxy_mask(42, 0, st, d, m, n)

    def check_xor():
        torch.cuda.synchronize()
        assert comm.poll() == 0, ppc.STATUS[comm.poll()]
        if rank in (0, S - 1):
            for m in range(M):
                y, g = xor_closed_form(S, m, P.source_activation(42, 0, m, n),
                                       P.source_gradient(42, 0, m, n), mask)
                assert np.array_equal(host(out[m])[:n], y if rank == S - 1 else g), (rank, m)
                out[m].fill_(0)

    ppc.step_1f1b(comm, xargs, s)
    check_xor()
    dist.barrier()
    graph = ppc.StepGraph([comm], [xargs], [s])
    for it in range(4):
        graph.launch()
        check_xor()
        if it == 1:
            ppc.step_1f1b(comm, xargs, s)      # eager step between graph launches
            check_xor()
    graph.destroy()
    # identity step with registered sources: zero-copy pulls captured in the graph
    ppc.register_tensors(comm, X or G)
    iargs = ppc.StepArgs(M, n, n, x=X, g=G, y=out if rank == S - 1 else None,
                         dx=out if rank == 0 else None)
    ppc.step_1f1b(comm, iargs, s)
    torch.cuda.synchronize()
    dist.barrier()
    g2 = ppc.StepGraph([comm], [iargs], [s])
    for _ in range(3):
        g2.launch()
        torch.cuda.synchronize()
        assert comm.poll() == 0
        if rank in (0, S - 1):
            for m in range(M):
                ref = P.source_gradient(42, 0, m, n) if rank == 0 else P.source_activation(42, 0, m, n)
                assert np.array_equal(host(out[m])[:n], ref), (rank, m)
                out[m].fill_(0)
    g2.destroy()
    return comm


def case_fullsize(rank, world):
    """BASELINE.json full sizes in bench.py's launch configuration (zero-copy registered
    sends, 256 KiB grain, the step replayed as a CUDA graph): 2 ranks = C2 (LLaMA-8B-shaped
    [1,4096,4096] bf16, PP=2, M=8); 4 ranks = C4 stand-in (Qwen2-7B-shaped [1,4096,3584],
    PP=4, M=32).  Identity stages: the last stage must hold X_m, stage 0 G_m, byte for byte;
    micro-batches 0, 1 and M-1 are compared (sampled), every step of 3 graph launches."""
    S = world
    hidden, M = (4096, 8) if world == 2 else (3584, 32)
    n = 4096 * hidden * 2
    cfg = ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=256 << 10)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    s = torch.cuda.Stream()
    X = [buf(n) for _ in range(M)] if rank == 0 else None
    G = [buf(n) for _ in range(M)] if rank == S - 1 else None
    out = [buf(n) for _ in range(M)] if rank in (0, S - 1) else None
    for m in range(M):
        if X:
            ppc.fill_payload(X[m], n, 42, 0, P.SRC_BOUNDARY, 0, m)
        if G:
            ppc.fill_payload(G[m], n, 42, 0, P.SRC_BOUNDARY, 1, m)
    ppc.register_tensors(comm, X or G or [])
    args = ppc.StepArgs(M, n, n, x=X, g=G, y=out if rank == S - 1 else None,
                        dx=out if rank == 0 else None)
    ppc.step_1f1b(comm, args, s)
    torch.cuda.synchronize()
    graph = ppc.StepGraph([comm], [args], [s])
    for _ in range(3):
        graph.launch()
        torch.cuda.synchronize()
        assert comm.poll() == 0
        if out:
            for m in (0, 1, M - 1):
                ref = P.source_gradient(42, 0, m, n) if rank == 0 else P.source_activation(42, 0, m, n)
                assert np.array_equal(host(out[m]), ref), (rank, m)
                out[m].fill_(0)
    graph.destroy()
    return comm


def case_gather(rank, world):
    """NEXT-1 TP-sliced boundary with a fused all-gather, PP=2 x TP=2 on 4 GPUs: each TP rank
    sends only its half of the boundary tensor; each TP rank of the other stage receives the
    whole tensor (both halves pulled over NVLink).  Compared byte for byte with the oracle's
    definition (concatenation of the TP slices = the full tensor), both directions, ragged."""
    from oracle.collectives import tp_gather_reference
    tp = 2
    cfg = ppc.make_config(tp=tp, pp=world // tp, dp=1, max_msg_bytes=4 << 20, chunk_bytes=256 << 10)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    s = torch.cuda.current_stream()
    pp_i, tp_i = rank // tp, rank % tp
    slice_n = 3 * (256 << 10) + 77
    total = tp * slice_n
    M = 3
    fulls = [buf(total) for _ in range(M)]           # what this rank sends slices of
    d_send = ppc.FWD if pp_i == 0 else ppc.BWD
    d_recv = ppc.BWD if pp_i == 0 else ppc.FWD
    for m in range(M):
        ppc.fill_payload(fulls[m], total, 42, 0, P.SRC_BOUNDARY, d_send, m)
    ppc.register_tensors(comm, fulls)
    outs = [buf(total) for _ in range(M)]
    # zero-copy sends complete on consumption: sends and gathers on two non-default streams
    # (the legacy default stream would serialise the gather behind the pending send)
    s_send = torch.cuda.Stream()
    s = torch.cuda.Stream()
    for m in range(M):
        comm.send(d_send, fulls[m].data_ptr() + tp_i * slice_n, slice_n, mb=m, stream=s_send)
        comm.recv_gather(d_recv, outs[m], total, mb=m, stream=s)
    torch.cuda.synchronize()
    assert comm.poll() == 0, comm.error_info()
    for m in range(M):
        full = P.payload_bytes(42, 0, P.SRC_BOUNDARY, d_recv, m, total)
        ref = tp_gather_reference([full[t * slice_n:(t + 1) * slice_n] for t in range(tp)])
        assert np.array_equal(host(outs[m]), ref), (rank, m)
    return comm


def case_hetero(rank, world):
    """NEXT-2: hetero allreduce = NCCL in each stage's DP subgroup + leader exchange over the
    PP path + NCCL broadcast; compared exactly (integer-valued fp32) with the oracle."""
    from oracle.collectives import allreduce_reference
    dp = 2 if world >= 4 else 1
    pp = world // dp
    cfg = ppc.make_config(tp=1, pp=pp, dp=dp, max_msg_bytes=8 << 20)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=True)
    n = (1 << 20) + 3
    idx = np.arange(n, dtype=np.int64)
    vals = {r: ((r + 1) * (idx % 7 + 1)).astype(np.float32) for r in range(world)}
    ref = allreduce_reference(vals, list(range(world)))
    for dtype, torch_dt in ((7, torch.float32), (2, torch.int32)):
        t = torch.from_numpy(vals[rank]).to(torch_dt).cuda()
        comm.hetero_allreduce(t, dtype, stream=torch.cuda.current_stream())
        torch.cuda.synchronize()
        assert comm.poll() == 0
        assert np.array_equal(t.cpu().numpy().astype(np.float64), ref), (rank, dtype)
    return comm


def case_inplace(rank, world, M=6):
    """Produce-in-place sends along a PP=world chain, both directions: every stage computes
    the XOR proxy of what it received straight into the next stage's ring slot — even mb
    with the fused kernel (per-chunk flags from the producer, ppc_stage_xor_send), odd mb
    with ppc_stage_xor writing into the slot and ppc_pp_send_end releasing the flags."""
    import ctypes as C
    S, n = world, 5 * (256 << 10) + 777
    cfg = ppc.make_config(pp=S, max_msg_bytes=n, chunk_bytes=256 << 10)
    comm = ppc.connect_distributed(cfg, rank, world, dev(rank), with_nccl=False)
    s = torch.cuda.current_stream()
    xor = ppc._lib.ppc_stage_xor
    xor.restype = C.c_int
    xor.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_size_t,
                    C.c_void_p]
    mask = lambda st, d, m: P.proxy_mask(42, 0, st, d, m, n)

    def forward(d, m, inp):
        ctx = ppc.XorCtx(42, 0, rank, d)
        if m % 2 == 0:
            comm.xor_send(d, ctx, m, inp, n, stream=s)
        else:
            sl = comm.send_begin(d, n, m, stream=s)
            assert xor(C.byref(ctx), m, inp.data_ptr(), sl.payload, n, n, s.cuda_stream) == 0
            comm.send_end(d, False, stream=s)

    for m in range(M):
        for d in (ppc.FWD, ppc.BWD):
            first = 0 if d == ppc.FWD else S - 1
            last = S - 1 if d == ppc.FWD else 0
            x = buf(n)
            if rank == first:
                ppc.fill_payload(x, n, 42, 0, 0, d, m, stream=s)
            else:
                comm.recv(d, x, n, mb=m, stream=s)
            if rank != last:
                forward(d, m, x)
            else:
                want = P.payload_bytes(42, 0, 0, d, m, n)
                for st in (range(S - 1) if d == ppc.FWD else range(S - 1, 0, -1)):
                    want = want ^ mask(st, d, m)
                assert np.array_equal(host(x)[:n], want), (rank, d, m)
    torch.cuda.synchronize()
    assert comm.poll() == 0
    return comm


CASES = {
    "sendrecv_sm": lambda r, w: case_sendrecv(r, w, ppc.ENGINE_SM),
    "sendrecv_ce": lambda r, w: case_sendrecv(r, w, ppc.ENGINE_CE),
    "sendrecv_pull": lambda r, w: case_sendrecv(r, w, ppc.ENGINE_PULL),
    "xor_sm": lambda r, w: case_xor(r, w, ppc.ENGINE_SM),
    "xor_ce": lambda r, w: case_xor(r, w, ppc.ENGINE_CE),
    "xor_pull": lambda r, w: case_xor(r, w, ppc.ENGINE_PULL),
    "timeout": case_timeout,
    "toy": case_toy,
    "hetero": case_hetero,
    "zc": case_zc,
    "zc_bidir_stream": case_zc_bidir_stream,
    "host": case_host,
    "zc_async": case_zc_async,
    "graph": case_graph,
    "inplace": case_inplace,
    "fullsize": case_fullsize,
    "gather": case_gather,
    "dcbs": case_dcbs,
    "dcbs1": case_dcbs1,
}
# cases that are another case under an environment setting
VARIANTS = {
    "zc_unfused": ("zc", {"PPC_FUSE_PUBLISH": "0"}),       # publication by its own kernel
    "zc_side": ("zc", {"PPC_ZC_SIDE": "1"}),               # publication on the send stream
    "xor_inplace": ("xor_sm", {"PPC_STEP_INPLACE": "1"}),  # stage fns produce into the slot
}


def run_case(case, rank, world):
    """One case end to end: its comm is disconnected and destroyed before returning."""
    if case in VARIANTS:
        base, env = VARIANTS[case]
        os.environ.update(env)
        case = base
    if case not in CASES:
        raise SystemExit(f"unknown case {case}")
    comm = CASES[case](rank, world)
    torch.cuda.synchronize()
    dist.barrier()
    comm.disconnect()
    dist.barrier()
    comm.destroy()


def main():
    """mp_worker.py CASE  |  mp_worker.py --batch JSON  (JSON = [[case, {env}], ...]: the
    cases run one after another in this process group, each with its environment set and
    the process environment restored afterwards; '#i case OK' per case)."""
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(dev(rank))
    dist.init_process_group("gloo")
    if sys.argv[1] == "--batch":
        import json
        import traceback
        for i, (case, env) in enumerate(json.loads(sys.argv[2])):
            saved = dict(os.environ)
            os.environ.update(env)
            try:
                run_case(case, rank, world)
            except BaseException:
                print(f"rank {rank} #{i} {case} FAIL", flush=True)
                traceback.print_exc()
                sys.stdout.flush()
                os._exit(1)               # the other ranks may be inside a collective
            finally:
                for k in set(os.environ) - set(saved):
                    del os.environ[k]
                os.environ.update(saved)
            print(f"rank {rank} #{i} {case} OK", flush=True)
    else:
        case = sys.argv[1]
        run_case(case, rank, world)
        print(f"rank {rank} {case} OK", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
