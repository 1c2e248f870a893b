"""C1 toy pipeline on the GPU (BASELINE.json configs[0]): a 2-stage x 2-layer MLP whose
boundary activations and gradients travel through libppc, compared with the oracle
(oracle/toy.py, fp64).  Gates (BJ north_star): loss within 1e-3 relative of the oracle (bf16
boundary and fp32 boundary); GPU pipelined == GPU un-pipelined bitwise (same kernels, same
per-stage order)."""
import numpy as np
import pytest
import torch

import paper_2602_18007_b200 as ppc
from oracle import toy as otoy
from synth.toy import ROWS, WIDTH, data, init_params

pytestmark = pytest.mark.gpu

M, LR, STEPS = 4, 10.0, 8


def _stages(bf16, devices):
    from paper_2602_18007_b200.toy import ToyStage
    Ws, bs = init_params(42)
    X, T = data(M, 42)
    s0 = ToyStage(0, ROWS, WIDTH, M, LR, bf16, devices[0], Ws[0:2], bs[0:2], X)
    s1 = ToyStage(1, ROWS, WIDTH, M, LR, bf16, devices[1], Ws[2:4], bs[2:4], T)
    return s0, s1


def run_pipelined(bf16, devices=(0, 0), steps=STEPS):
    s0, s1 = _stages(bf16, devices)
    cfg = ppc.make_config(pp=2, max_msg_bytes=s0.boundary_bytes, chunk_bytes=64 << 10)
    comms = ppc.virtual_stages(cfg, list(devices))
    streams = [torch.cuda.Stream(device=d) for d in devices]
    args = [s0.step_args(), s1.step_args()]
    losses = []
    for _ in range(steps):
        ppc.step_1f1b_local(comms, args, streams)
        losses.append(s1.loss(streams[1]))
        s0.step_end(streams[0])
        s1.step_end(streams[1])
    params = s0.params() + s1.params()
    for c in comms:
        assert c.poll() == 0
        c.disconnect()
    for c in comms:
        c.destroy()
    s0.destroy()
    s1.destroy()
    return losses, params


def run_unpipelined(bf16, steps=STEPS):
    """Same kernels, one stream, no transfers: all F_m then all B_m ascending."""
    s0, s1 = _stages(bf16, (0, 0))
    nb = s0.boundary_bytes
    act = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(M)]
    grd = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(M)]
    s = torch.cuda.current_stream()
    losses = []
    for _ in range(steps):
        for m in range(M):
            s0.fwd(m, None, act[m].data_ptr(), s)
            s1.fwd(m, act[m].data_ptr(), None, s)
        for m in range(M):
            s1.bwd(m, None, grd[m].data_ptr(), s)
            s0.bwd(m, grd[m].data_ptr(), None, s)
        losses.append(s1.loss(s))
        s0.step_end(s)
        s1.step_end(s)
    params = s0.params() + s1.params()
    s0.destroy()
    s1.destroy()
    return losses, params


def oracle_series(bf16, steps=STEPS):
    Ws, bs = init_params(42)
    X, T = data(M, 42)
    series, W, B = otoy.train(Ws, bs, X, T, steps, lr=LR, dtype=np.float64, bf16=bf16)
    return series, W, B


@pytest.mark.parametrize("bf16", [False, True])
def test_toy_loss_matches_oracle(bf16):
    gpu, (W0, b0, W1, b1) = run_pipelined(bf16)
    ref, Wr, Br = oracle_series(bf16)
    rel = max(abs(g - r) / abs(r) for g, r in zip(gpu, ref))
    assert rel <= 1e-3, (gpu, ref)
    assert all(b < a for a, b in zip(gpu, gpu[1:]))
    Wg = [W0[0], W0[1], W1[0], W1[1]]
    for wg, wr in zip(Wg, Wr):
        assert np.linalg.norm(wg - wr) <= 1e-3 * np.linalg.norm(wr)


@pytest.mark.parametrize("bf16", [False, True])
def test_toy_pipelined_equals_unpipelined_bitwise(bf16):
    lp, pp_ = run_pipelined(bf16)
    lu, pu = run_unpipelined(bf16)
    assert lp == lu
    for a, b in zip(pp_, pu):
        assert np.array_equal(a, b)


def test_toy_across_two_gpus_in_one_process():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    l2, p2 = run_pipelined(True, devices=(0, 1))
    l1, p1 = run_pipelined(True, devices=(0, 0))
    assert l2 == l1                      # same kernels, same order: bitwise across devices
    for a, b in zip(p2, p1):
        assert np.array_equal(a, b)
