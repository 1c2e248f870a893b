"""O5 — a 1F1B step executed byte for byte over O3 channels, with a stage function.
TEST INFRASTRUCTURE ONLY.

The step follows O1's per-stage op order and the dependency
rules of O2: F_m at stage s receives FWD m from s-1 (s > 0), applies the stage
function, sends FWD m to s+1 (s < S-1); B_m receives BWD m from s+1 (s < S-1),
applies the backward stage function, sends BWD m to s-1 (s > 0).  Stages are
interleaved by a plain round-robin executor: any stage whose next op has its
message available (and, for its send, a free slot) runs it.  Every dependency-
respecting interleaving gives the same bytes; the executor records the one it used.

Integer stage proxy (schedule-order witness, R9): F at stage s is
y = x XOR H_F(s, m), B at stage s is g' = g XOR H_B(s, m), bytewise, with the masks
passed in as inputs (synth/payload.proxy_mask).  Closed form after one step:
    Y_m  = X_m XOR H_F(0,m) XOR ... XOR H_F(S-1,m)          (last stage, forward)
    dX_m = G_m XOR H_B(S-1,m) XOR ... XOR H_B(0,m)          (stage 0, backward)
so any dropped, duplicated, swapped or mis-delivered message changes the result.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Optional, Tuple

import numpy as np

from .schedule import schedule_1f1b
from .transfer import BWD, FWD, Channel, WouldBlock, make_channels

StageFn = Callable[[int, int, np.ndarray], np.ndarray]


def run_1f1b(S: int, M: int, K: int, fwd: StageFn, bwd: StageFn,
             src: Callable[[int], np.ndarray], dsrc: Callable[[int], np.ndarray],
             max_bytes: int, fwd_bytes: int, bwd_bytes: int):
    """Run one step.  `src(m)`: stage-0 input of F_m; `dsrc(m)`: stage S-1 input of B_m.
    Receivers expect `fwd_bytes` / `bwd_bytes` per message (their tensor size).
    Returns (Y, dX, channels, order): last-stage forward outputs, stage-0 backward
    outputs, the O3 channels (with their delivery logs) and the executed op order."""
    chans = make_channels(S, K, max_bytes)
    orders = [schedule_1f1b(S, s, M) for s in range(S)]
    idx = [0] * S
    Y: Dict[int, np.ndarray] = {}
    dX: Dict[int, np.ndarray] = {}
    pending: List[Optional[Tuple[Channel, np.ndarray, int]]] = [None] * S  # send blocked on a slot
    order: List[Tuple[int, str, int]] = []
    total = sum(len(o) for o in orders)
    done = 0
    while done < total or any(p is not None for p in pending):
        moved = False
        for s in range(S):
            if pending[s] is not None:
                ch, data, m = pending[s]
                try:
                    ch.send(data, m)
                    pending[s] = None
                    moved = True
                except WouldBlock:
                    continue
            if idx[s] >= len(orders[s]):
                continue
            kind, m = orders[s][idx[s]]
            if kind == "F":
                if s > 0:
                    ch_in = chans[(FWD, s - 1)]
                    if ch_in.send_seq < ch_in.recv_seq + 1:
                        continue
                    x = ch_in.recv(fwd_bytes, m)
                else:
                    x = src(m)
                y = fwd(s, m, x)
                if s < S - 1:
                    pending[s] = (chans[(FWD, s)], y, m)
                else:
                    Y[m] = y
            else:
                if s < S - 1:
                    ch_in = chans[(BWD, s)]
                    if ch_in.send_seq < ch_in.recv_seq + 1:
                        continue
                    g = ch_in.recv(bwd_bytes, m)
                else:
                    g = dsrc(m)
                g2 = bwd(s, m, g)
                if s > 0:
                    pending[s] = (chans[(BWD, s - 1)], g2, m)
                else:
                    dX[m] = g2
            idx[s] += 1
            done += 1
            order.append((s, kind, m))
            moved = True
            if pending[s] is not None:
                ch, data, mm = pending[s]
                try:
                    ch.send(data, mm)
                    pending[s] = None
                except WouldBlock:
                    pass
        if not moved:
            raise RuntimeError(f"byte-level 1F1B run stuck at idx={idx}")
    return Y, dX, chans, order


def xor_stage(masks: Callable[[int, int, int], np.ndarray], direction: int) -> StageFn:
    """F (direction 0) / B (direction 1) stage proxy: x XOR mask(stage, direction, m)."""
    def fn(s: int, m: int, x: np.ndarray) -> np.ndarray:
        return np.bitwise_xor(x, masks(s, direction, m))
    return fn


def xor_closed_form(S: int, m: int, x0: np.ndarray, g0: np.ndarray,
                    masks: Callable[[int, int, int], np.ndarray]):
    """Y_m and dX_m by XOR algebra (no pipeline)."""
    y = x0.copy()
    for s in range(S):
        y ^= masks(s, FWD, m)
    g = g0.copy()
    for s in reversed(range(S)):
        g ^= masks(s, BWD, m)
    return y, g
