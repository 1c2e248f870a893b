"""Inputs of the C1 toy pipeline (BASELINE.json configs[0]): initial weights, data, targets.

Recipe (ambiguity A11):
  * r = numpy.random.default_rng(seed); W0..W3 = r.uniform(-1/16, 1/16, (256, 256)) in
    that order, then b0..b3 = r.uniform(-1/16, 1/16, (256,)).  1/16 = 1/sqrt(fan_in).
  * A separate default_rng(seed) draws X_0..X_{M-1} = standard_normal((128, 256)).
  * A = default_rng(seed + 1).standard_normal((256, 256)) / 16; T_m = X_m @ A.
All draws are float64; callers cast to their working dtype.
"""
from __future__ import annotations

import numpy as np

WIDTH = 256      # boundary hidden size, BASELINE.json configs[0] "[1,128,256]"
ROWS = 128       # sequence length of the toy boundary tensor
N_LAYERS = 4     # 2 stages x 2 layers ("2-layer MLP per stage")


def init_params(seed: int = 42):
    r = np.random.default_rng(seed)
    lim = 1.0 / 16.0
    Ws = [r.uniform(-lim, lim, (WIDTH, WIDTH)) for _ in range(N_LAYERS)]
    bs = [r.uniform(-lim, lim, (WIDTH,)) for _ in range(N_LAYERS)]
    return Ws, bs


def data(M: int = 4, seed: int = 42):
    r = np.random.default_rng(seed)
    X = [r.standard_normal((ROWS, WIDTH)) for _ in range(M)]
    A = np.random.default_rng(seed + 1).standard_normal((WIDTH, WIDTH)) / 16.0
    T = [x @ A for x in X]
    return X, T
