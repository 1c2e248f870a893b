"""Heterogeneous-collective composition.  TEST INFRASTRUCTURE ONLY.

PAPER.md §2.2: "each homogeneous subgroup ... first performs intra-group aggregation
using its vendor-specific CCL. Subsequently, the CPU-offloading P2P mechanism transfers these
intermediate results across the heterogeneous cluster to achieve global collective
communication synchronization".  SPEC.md S:L423-446: the result equals a single-process
reduction over all ranks (exact for integers).

`allreduce_reference` is that plain definition: for every rank, the sum over all ranks of
its group, in ascending rank order (float64).  `composed_allreduce` follows the paper's
three phases literally (subgroup sums, leader exchange along the stage chain, subgroup
broadcast) so a test can check the composition reproduces the plain definition.

Pins (tests/test_oracle_collectives.py): SPEC worked examples — allreduce of rank ids over
4 ranks -> 6; hetero allreduce {1,2 | 3,4} -> 10.
"""
from __future__ import annotations

from typing import Dict, List

import numpy as np

from .groups import build_groups, coords


def allreduce_reference(values: Dict[int, np.ndarray], group: List[int]) -> np.ndarray:
    acc = np.zeros_like(np.asarray(values[group[0]], dtype=np.float64))
    for r in sorted(group):
        acc = acc + np.asarray(values[r], dtype=np.float64)
    return acc


def composed_allreduce(values: Dict[int, np.ndarray], world: int, tp: int, pp: int, dp: int):
    """Per rank result of the 3-phase composition over the ranks sharing tp_i: subgroups =
    each stage's DP group; leaders = dp_i 0, chained along the PP stages."""
    out = {}
    for t in range(tp):
        ranks = [r for r in range(world) if coords(r, tp, pp, dp)[2] == t]
        sub = {}                                   # phase 1: per-stage subgroup sums
        for r in ranks:
            p = coords(r, tp, pp, dp)[0]
            sub.setdefault(p, []).append(r)
        partial = {p: allreduce_reference(values, g) for p, g in sub.items()}
        total = np.zeros_like(partial[0])          # phase 2: leader chain, forward
        for p in range(pp):
            total = total + partial[p]
        for r in ranks:                            # phase 3: broadcast inside subgroups
            out[r] = total.copy()
    return out


def tp_gather_reference(slices):
    """TP-sliced boundary: the receiving stage's tensor is the
    concatenation of the sending TP ranks' slices in tp order (an all-gather)."""
    return np.concatenate([np.asarray(x) for x in slices])


def groups_for(world: int, tp: int, pp: int, dp: int):
    return build_groups(world, tp, pp, dp)
