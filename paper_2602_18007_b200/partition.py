"""Uneven layer partition of a PP pipeline from measured per-layer times.

PAPER.md §4.2: "we adopt an uneven partitioning scheme, assigning fewer
Transformer layers to the AMD GPUs due to their lower observed throughput ... Under a proper
partitioning strategy, the expected performance satisfies AMD < AMD+NVIDIA < NVIDIA";
§3.1.2 gives the splits (LLaMA-8B 16-16 homogeneous, 15-17 heterogeneous).

Host-side planning (no GPU): `iteration_time` runs a compact event model of one
non-interleaved 1F1B step (per-stage op order from libppc's ppc_schedule_1f1b; a message
arrives `comm_us` after its producing op ends; sends are asynchronous), and
`optimize_partition` searches every composition of the layers (exhaustive, fine for the
paper's PP = 2 and small PP), breaking ties toward the most even split.
"""
from __future__ import annotations

import itertools
from typing import List, Optional, Sequence

from . import schedule_1f1b


def iteration_time(layers: Sequence[int], t_fwd: Sequence[float], t_bwd: Sequence[float], M: int,
                   comm_us: float = 0.0, extra_fwd: Optional[Sequence[float]] = None,
                   extra_bwd: Optional[Sequence[float]] = None) -> float:
    """Step time of a 1F1B pipeline: stage s runs layers[s] layers of per-layer time
    t_fwd[s] / t_bwd[s] (+ optional fixed per-micro-batch extra, e.g. embedding / LM head)."""
    S = len(layers)
    f = [layers[s] * t_fwd[s] + (extra_fwd[s] if extra_fwd else 0.0) for s in range(S)]
    b = [layers[s] * t_bwd[s] + (extra_bwd[s] if extra_bwd else 0.0) for s in range(S)]
    ops = [schedule_1f1b(S, s, M) for s in range(S)]
    idx = [0] * S
    free = [0.0] * S
    end_f = {}
    end_b = {}
    done = 0
    total = 2 * S * M
    while done < total:
        moved = False
        for s in range(S):
            while idx[s] < len(ops[s]):
                kind, m = ops[s][idx[s]]
                if kind == "F":
                    dep = end_f.get((s - 1, m)) if s > 0 else 0.0
                    if dep is None:
                        break
                    start = max(free[s], dep + (comm_us if s > 0 else 0.0))
                    end_f[(s, m)] = free[s] = start + f[s]
                else:
                    dep = end_b.get((s + 1, m)) if s < S - 1 else end_f[(s, m)]
                    if dep is None:
                        break
                    start = max(free[s], dep + (comm_us if s < S - 1 else 0.0))
                    end_b[(s, m)] = free[s] = start + b[s]
                idx[s] += 1
                done += 1
                moved = True
        if not moved:
            raise RuntimeError("1F1B model made no progress")
    return max(free)


def _compositions(total: int, parts: int):
    for cuts in itertools.combinations(range(1, total), parts - 1):
        edges = (0,) + cuts + (total,)
        yield [edges[i + 1] - edges[i] for i in range(parts)]


def optimize_partition(total_layers: int, t_fwd: Sequence[float], t_bwd: Sequence[float], M: int,
                       comm_us: float = 0.0, extra_fwd=None, extra_bwd=None) -> List[int]:
    """Layers per stage minimising iteration_time; ties -> the most even split."""
    S = len(t_fwd)
    if total_layers < S:
        raise ValueError("Infeasible: fewer layers than stages")
    best, best_key = None, None
    for comp in _compositions(total_layers, S):
        t = iteration_time(comp, t_fwd, t_bwd, M, comm_us, extra_fwd, extra_bwd)
        key = (round(t, 9), max(comp) - min(comp))
        if best_key is None or key < best_key:
            best, best_key = comp, key
    return best
