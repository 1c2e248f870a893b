"""O6 — the C1 toy pipeline: 2 stages x 2 layers MLP, MSE loss, SGD.  TEST INFRASTRUCTURE ONLY.

Follows SPEC.md trainer (dense layers, mean squared error, seeded
initialiser, SGD with fixed learning rate, fixed evaluation order, fp64, pipelined
== single-process bitwise) and BASELINE.json configs[0] (boundary [1,128,256] fp32,
2-layer MLP per stage, 4 micro-batches), in the reading DESIGN.md R11 fixes:
  layer l (l = 0..3): z_l = h_l @ W_l + b_l ; h_{l+1} = tanh(z_l) for l < 3, Y = z_3
  stage 0 holds layers 0, 1 and sends the boundary a = h_2 (FWD); stage 1 holds
  layers 2, 3 and sends back dL/da (BWD).
  L = (1/M) sum_m mean((Y_m - T_m)^2)                    (R10)
  dL/dY_m = 2 (Y_m - T_m) / (128 * 256 * M)
  weight gradients accumulate over m in ascending order starting from zero;
  SGD at the end of the step: p -= lr * grad (lr = 10, R11).
Optional bf16 boundary (O7): the boundary tensor and its gradient are rounded
through bf16 before they are sent.

Pinned by tests/test_oracle_toy.py: pipelined (through O3 channels, O1 order) ==
un-pipelined bitwise in fp64 and fp32; central finite differences; torch.autograd
in CPU fp64 (library special case) on the same MLP; monotone loss decrease.
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np

from . import bf16 as _bf16
from .proxy import run_1f1b

ROWS, WIDTH = 128, 256


def _layer_fwd(W, b, h, act: bool):
    z = h @ W + b
    return np.tanh(z) if act else z


def stage0_forward(W, B, x):
    """Layers 0, 1.  Returns boundary a = tanh(tanh(x W0 + b0) W1 + b1) and the cache."""
    h1 = _layer_fwd(W[0], B[0], x, True)
    a = _layer_fwd(W[1], B[1], h1, True)
    return a, (x, h1, a)


def stage1_forward(W, B, a):
    """Layers 2, 3 (last linear).  Returns Y and the cache."""
    h3 = _layer_fwd(W[2], B[2], a, True)
    y = _layer_fwd(W[3], B[3], h3, False)
    return y, (a, h3, y)


def loss_m(y, t):
    return np.mean((y - t) ** 2)


def stage1_backward(W, cache, t, M):
    """dL/dY -> grads of layers 2, 3 and dL/da."""
    a, h3, y = cache
    dt = y.dtype
    dy = (2.0 * (y - t) / dt.type(ROWS * WIDTH * M)).astype(dt)
    gW3 = h3.T @ dy
    gb3 = dy.sum(axis=0)
    dh3 = dy @ W[3].T
    dz2 = dh3 * (1 - h3 * h3)
    gW2 = a.T @ dz2
    gb2 = dz2.sum(axis=0)
    da = dz2 @ W[2].T
    return da, (gW2, gb2, gW3, gb3)


def stage0_backward(W, cache, da):
    x, h1, a = cache
    dz1 = da * (1 - a * a)
    gW1 = h1.T @ dz1
    gb1 = dz1.sum(axis=0)
    dh1 = dz1 @ W[1].T
    dz0 = dh1 * (1 - h1 * h1)
    gW0 = x.T @ dz0
    gb0 = dz0.sum(axis=0)
    return (gW0, gb0, gW1, gb1)


def _cast_params(Ws, bs, dtype):
    return [np.array(w, dtype=dtype) for w in Ws], [np.array(b, dtype=dtype) for b in bs]


def _boundary(x, bf16: bool):
    return _bf16.round_through_bf16(x) if bf16 else x


def unpipelined_step(W, B, X, T, lr, bf16=False):
    """Reference: the same per-micro-batch functions in one process, m ascending.
    Returns (loss, W', B')."""
    M = len(X)
    dt = W[0].dtype
    g = [np.zeros_like(W[i]) for i in range(4)] + [np.zeros_like(B[i]) for i in range(4)]
    loss = dt.type(0)
    caches0, caches1 = [], []
    for m in range(M):               # F_m (order of forwards is irrelevant to the math)
        a, c0 = stage0_forward(W, B, X[m])
        a = _boundary(a, bf16)
        y, c1 = stage1_forward(W, B, a)
        caches0.append(c0)
        caches1.append(c1)
    for m in range(M):
        loss = loss + loss_m(caches1[m][2], T[m]) / dt.type(M)
    for m in range(M):               # B_m ascending; accumulation order fixed
        da, (gW2, gb2, gW3, gb3) = stage1_backward(W, caches1[m], T[m], M)
        da = _boundary(da, bf16)
        gW0, gb0, gW1, gb1 = stage0_backward(W, caches0[m], da)
        for i, v in zip((0, 1, 2, 3), (gW0, gW1, gW2, gW3)):
            g[i] = g[i] + v
        for i, v in zip((0, 1, 2, 3), (gb0, gb1, gb2, gb3)):
            g[4 + i] = g[4 + i] + v
    W2 = [W[i] - dt.type(lr) * g[i] for i in range(4)]
    B2 = [B[i] - dt.type(lr) * g[4 + i] for i in range(4)]
    return loss, W2, B2


def pipelined_step(W, B, X, T, lr, bf16=False, K=2):
    """The same step executed as a 2-stage 1F1B pipeline whose boundary tensors
    travel as bytes through O3 channels (O5's executor).  Returns (loss, W', B', order)."""
    M = len(X)
    dt = W[0].dtype
    state: Dict[Tuple[int, int], tuple] = {}
    grads = {s: None for s in (0, 1)}
    losses: List = [None] * M

    def to_bytes(a):
        a = _boundary(a, bf16)
        if bf16:
            return _bf16.f32_to_bf16_bits(a.astype(np.float32)).view(np.uint8).reshape(-1).copy()
        return np.ascontiguousarray(a).view(np.uint8).reshape(-1).copy()

    def from_bytes(raw):
        if bf16:
            return _bf16.bf16_bits_to_f32(raw.view(np.uint16)).astype(dt).reshape(ROWS, WIDTH)
        return raw.view(dt).reshape(ROWS, WIDTH).copy()

    def fwd(s, m, x):
        if s == 0:
            a, c = stage0_forward(W, B, X[m])
            state[(0, m)] = c
            return to_bytes(a)
        y, c = stage1_forward(W, B, from_bytes(x))
        state[(1, m)] = c
        losses[m] = loss_m(y, T[m])
        return np.zeros(0, np.uint8)

    def acc(s, vals):
        if grads[s] is None:
            grads[s] = [np.zeros_like(v) for v in vals]
        grads[s] = [gacc + v for gacc, v in zip(grads[s], vals)]

    def bwd(s, m, g):
        if s == 1:
            da, gl = stage1_backward(W, state[(1, m)], T[m], M)
            acc(1, gl)
            return to_bytes(da)
        gl = stage0_backward(W, state[(0, m)], from_bytes(g))
        acc(0, gl)
        return np.zeros(0, np.uint8)

    nb = ROWS * WIDTH * (2 if bf16 else dt.itemsize)
    _, _, chans, order = run_1f1b(2, M, K, fwd, bwd, src=lambda m: None,
                                  dsrc=lambda m: None, max_bytes=nb, fwd_bytes=nb, bwd_bytes=nb)
    loss = dt.type(0)
    for m in range(M):
        loss = loss + losses[m] / dt.type(M)
    gW0, gb0, gW1, gb1 = grads[0]
    gW2, gb2, gW3, gb3 = grads[1]
    g = [gW0, gW1, gW2, gW3, gb0, gb1, gb2, gb3]
    W2 = [W[i] - dt.type(lr) * g[i] for i in range(4)]
    B2 = [B[i] - dt.type(lr) * g[4 + i] for i in range(4)]
    return loss, W2, B2, order


def train(Ws, bs, X, T, steps, lr=10.0, dtype=np.float64, pipelined=False, bf16=False):
    """Loss series over `steps` steps (loss reported before each update)."""
    W, B = _cast_params(Ws, bs, dtype)
    Xc = [np.asarray(x, dtype=dtype) for x in X]
    Tc = [np.asarray(t, dtype=dtype) for t in T]
    series = []
    for _ in range(steps):
        if pipelined:
            loss, W, B, _ = pipelined_step(W, B, Xc, Tc, lr, bf16)
        else:
            loss, W, B = unpipelined_step(W, B, Xc, Tc, lr, bf16)
        series.append(float(loss))
    return series, W, B
