"""DCBS rank grid, parallel groups and backend assignment (§8(a) row a1).  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2.1 P:L42 (DCBS: "we employ the Gloo backend for inter-group PP
communication ... DP and TP groups remain homogeneous, continuing to leverage
vendor-specific libraries"), P:L47 ("differentiated initialization of
communication group backends") and §4.1 P:L198 ("we restrict heterogeneity to PP"),
with SPEC.md's grid: tp fastest, dp middle, pp slowest:
    rank = pp_i * (tp * dp) + dp_i * tp + tp_i
TP group = ranks sharing (pp_i, dp_i); DP group = sharing (pp_i, tp_i);
PP group = sharing (dp_i, tp_i), ordered by pp_i (stage order).
Backend: TP, DP -> "NCCL" (vendor CCL); PP -> "PEER" (the custom device-direct
kernels that replace the paper's CPU-offloading P2P).  Requesting the custom path
for a TP/DP group is a DCBS violation -> BackendError.

Pinned by tests/test_oracle_groups.py: SPEC's worked example (world 16, tp=1,
pp=2, dp=8 -> PP pairs (i, i+8)), partition invariants (every rank in
exactly one group of each kind, group sizes tp/dp/pp) and brute-force coordinate
enumeration.
"""
from __future__ import annotations

from typing import Dict, List, Tuple


class GridMismatch(ValueError):
    pass


class BackendError(ValueError):
    pass


def coords(rank: int, tp: int, pp: int, dp: int) -> Tuple[int, int, int]:
    """(pp_i, dp_i, tp_i) of `rank`."""
    if not (0 <= rank < tp * pp * dp):
        raise ValueError("rank out of range")
    return rank // (tp * dp), (rank % (tp * dp)) // tp, rank % tp


def rank_of(pp_i: int, dp_i: int, tp_i: int, tp: int, dp: int) -> int:
    return pp_i * (tp * dp) + dp_i * tp + tp_i


def build_groups(world: int, tp: int, pp: int, dp: int) -> Dict[str, List[List[int]]]:
    if min(tp, pp, dp) < 1 or tp * pp * dp != world:
        raise GridMismatch(f"tp*pp*dp = {tp * pp * dp} != world {world}")
    groups: Dict[str, List[List[int]]] = {"tp": [], "dp": [], "pp": []}
    for p in range(pp):
        for d in range(dp):
            groups["tp"].append([rank_of(p, d, t, tp, dp) for t in range(tp)])
    for p in range(pp):
        for t in range(tp):
            groups["dp"].append([rank_of(p, d, t, tp, dp) for d in range(dp)])
    for d in range(dp):
        for t in range(tp):
            groups["pp"].append([rank_of(p, d, t, tp, dp) for p in range(pp)])
    return groups


def group_of(rank: int, kind: str, world: int, tp: int, pp: int, dp: int) -> List[int]:
    for g in build_groups(world, tp, pp, dp)[kind]:
        if rank in g:
            return g
    raise AssertionError("unreachable")


def backend(kind: str, requested: str = "auto") -> str:
    native = {"tp": "NCCL", "dp": "NCCL", "pp": "PEER"}[kind]
    if requested == "auto":
        return native
    if requested == "PEER" and kind in ("tp", "dp"):
        raise BackendError("custom P2P path is for PP groups only (P:L198)")
    return requested


def pp_neighbors(rank: int, world: int, tp: int, pp: int, dp: int) -> Tuple[int, int]:
    """(previous stage rank or -1, next stage rank or -1) in this rank's PP group."""
    g = group_of(rank, "pp", world, tp, pp, dp)
    i = g.index(rank)
    return (g[i - 1] if i > 0 else -1, g[i + 1] if i < len(g) - 1 else -1)
