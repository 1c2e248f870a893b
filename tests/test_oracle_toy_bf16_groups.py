"""Pins for oracle O6 (toy pipeline), O7 (bf16 RNE) and the DCBS grid.

Pins: pipelined == un-pipelined bitwise, central finite differences within
1e-4 relative, torch.autograd in CPU fp64 on the same MLP (library special
case), loss ratio at step 200 < 0.1; torch CPU bf16 conversion; SPEC's
group-layout worked example.
"""
import numpy as np
import pytest
import torch

from oracle import bf16 as B16
from oracle import groups as G
from oracle import toy
from synth.toy import data, init_params


@pytest.fixture(scope="module")
def toy_inputs():
    Ws, bs = init_params(42)
    X, T = data(4, 42)
    return Ws, bs, X, T


@pytest.mark.parametrize("dtype,bf16", [(np.float64, False), (np.float32, False),
                                        (np.float32, True), (np.float64, True)])
def test_pipelined_equals_unpipelined_bitwise(toy_inputs, dtype, bf16):
    Ws, bs, X, T = toy_inputs
    s1, W1, B1 = toy.train(Ws, bs, X, T, 3, dtype=dtype, bf16=bf16)
    s2, W2, B2 = toy.train(Ws, bs, X, T, 3, dtype=dtype, bf16=bf16, pipelined=True)
    assert s1 == s2
    assert all(np.array_equal(a, b) for a, b in zip(W1 + B1, W2 + B2))


def _loss_and_grads(W, B, X, T):
    """One forward/backward with lr = 0 to read gradients: grad = (p - p') / lr is
    ill-posed, so call the stage functions directly."""
    M = len(X)
    g = [np.zeros_like(w) for w in W] + [np.zeros_like(b) for b in B]
    loss = 0.0
    for m in range(M):
        a, c0 = toy.stage0_forward(W, B, X[m])
        y, c1 = toy.stage1_forward(W, B, a)
        loss += toy.loss_m(y, T[m]) / M
        da, (gW2, gb2, gW3, gb3) = toy.stage1_backward(W, c1, T[m], M)
        gW0, gb0, gW1, gb1 = toy.stage0_backward(W, c0, da)
        for i, v in enumerate((gW0, gW1, gW2, gW3, gb0, gb1, gb2, gb3)):
            g[i] = g[i] + v
    return loss, g


def test_finite_differences(toy_inputs):
    Ws, bs, X, T = toy_inputs
    W = [w.copy() for w in Ws]
    B = [b.copy() for b in bs]
    _, g = _loss_and_grads(W, B, X, T)
    params = W + B
    rng = np.random.default_rng(3)
    h = 1e-5
    worst = 0.0
    for _ in range(10):
        i = int(rng.integers(0, 8))
        idx = tuple(int(rng.integers(0, n)) for n in params[i].shape)
        old = params[i][idx]
        params[i][idx] = old + h
        lp, _ = _loss_and_grads(W, B, X, T)
        params[i][idx] = old - h
        lm, _ = _loss_and_grads(W, B, X, T)
        params[i][idx] = old
        fd = (lp - lm) / (2 * h)
        an = g[i][idx]
        rel = abs(fd - an) / max(abs(fd), abs(an), 1e-12)
        worst = max(worst, rel)
    assert worst < 1e-4


def test_torch_autograd_library_case(toy_inputs):
    Ws, bs, X, T = toy_inputs
    _, g = _loss_and_grads([w.copy() for w in Ws], [b.copy() for b in bs], X, T)
    tw = [torch.tensor(w, dtype=torch.float64, requires_grad=True) for w in Ws]
    tb = [torch.tensor(b, dtype=torch.float64, requires_grad=True) for b in bs]
    loss = 0
    for x, t in zip(X, T):
        h = torch.tensor(x)
        for l in range(4):
            h = h @ tw[l] + tb[l]
            if l < 3:
                h = torch.tanh(h)
        loss = loss + torch.nn.functional.mse_loss(h, torch.tensor(t)) / len(X)
    loss.backward()
    ref = [p.grad.numpy() for p in tw + tb]
    for a, r in zip(g, ref):
        assert np.linalg.norm(a - r) <= 1e-12 * max(np.linalg.norm(r), 1e-30)


def test_training_converges(toy_inputs):
    Ws, bs, X, T = toy_inputs
    series, _, _ = toy.train(Ws, bs, X, T, 200)
    assert all(b < a for a, b in zip(series, series[1:]))     # monotone at lr 10
    assert series[-1] < 0.1 * series[0]
    # regression anchor (SURVEY App. A10 scratch run of this exact recipe; not a paper value)
    assert series[0] == pytest.approx(1.0033152624130217, rel=1e-15)


def test_bf16_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(200000).astype(np.float32),
        (rng.standard_normal(100000) * 1e-39).astype(np.float32),     # subnormals
        np.clip(rng.standard_normal(100000) * 3e38, -3.4e38, 3.4e38).astype(np.float32),
        np.array([0.0, -0.0, np.inf, -np.inf, 3.4028235e38, -3.4028235e38, 1.0, 1.00390625,
                  1.005859375, 1.001953125, 1.0078125 + 2 ** -8], dtype=np.float32),
    ])
    # exact ties: low 16 bits == 0x8000 with even and odd bit 16
    ties = (rng.integers(0, 1 << 15, 1000, dtype=np.uint32) << 17 | 0x8000).view(np.float32)
    ties2 = ((rng.integers(0, 1 << 15, 1000, dtype=np.uint32) << 17) | 0x18000).view(np.float32)
    x = np.concatenate([x, ties[np.isfinite(ties)], ties2[np.isfinite(ties2)]])
    ours = B16.f32_to_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    back = B16.bf16_bits_to_f32(ours)
    assert np.array_equal(back, torch.from_numpy(x).to(torch.bfloat16).float().numpy())
    nan = B16.f32_to_bf16_bits(np.array([np.nan], np.float32))
    assert np.isnan(B16.bf16_bits_to_f32(nan)).all()


def test_groups_spec_example():
    g = G.build_groups(16, tp=1, pp=2, dp=8)
    assert sorted(g["pp"]) == [[i, i + 8] for i in range(8)]
    assert all(len(x) == 1 for x in g["tp"])
    assert sorted(g["dp"]) == [list(range(8)), list(range(8, 16))]


@pytest.mark.parametrize("tp,pp,dp", [(1, 2, 1), (2, 4, 1), (1, 8, 1), (2, 2, 2), (3, 2, 2)])
def test_groups_partition(tp, pp, dp):
    world = tp * pp * dp
    g = G.build_groups(world, tp, pp, dp)
    for kind, size in (("tp", tp), ("pp", pp), ("dp", dp)):
        flat = sorted(r for grp in g[kind] for r in grp)
        assert flat == list(range(world))
        assert all(len(grp) == size for grp in g[kind])
    # brute force coordinates: rank <-> (pp_i, dp_i, tp_i) is a bijection, tp fastest
    seen = {}
    for r in range(world):
        c = G.coords(r, tp, pp, dp)
        assert G.rank_of(*c, tp, dp) == r
        seen[c] = r
    assert len(seen) == world
    for grp in g["pp"]:
        assert [G.coords(r, tp, pp, dp)[0] for r in grp] == list(range(pp))
    prev, nxt = G.pp_neighbors(0, world, tp, pp, dp)
    assert prev == -1 and nxt == tp * dp


def test_groups_errors():
    with pytest.raises(G.GridMismatch):
        G.build_groups(8, 2, 2, 1)
    with pytest.raises(G.BackendError):
        G.backend("tp", "PEER")
    assert G.backend("pp") == "PEER" and G.backend("dp") == "NCCL"
