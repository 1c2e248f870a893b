"""O1 — non-interleaved 1F1B op order for one pipeline stage.  TEST INFRASTRUCTURE ONLY.

Follows SPEC.md S:L577 ("Schedule = 1F1B (non-interleaved) with warmup =
min(pp - stage_index, microbatches)") in the reading DESIGN.md R2 fixes: warm-up
w = min(S - s - 1, M) forward ops, then M - w steady (F, B) pairs, then w
cool-down backward ops.  (SPEC's min(S - s, M) with (B, F) steady pairs yields the
identical sequence; tests/test_oracle_schedule.py checks that for S <= 8, M < 40.)
The paper itself never names its schedule (PAPER.md is silent; BJ north_star
names 1F1B).

Pinned by: brute-force enumeration of all in-flight-bounded per-stage orders
(1F1B is the unique makespan argmin under uniform costs), the zero-comm closed form
(M + S - 1)(f + b), SPEC's 1-stage case M(f + b), and op counting.
"""
from __future__ import annotations

from typing import List, Tuple

Op = Tuple[str, int]   # ("F" | "B", micro-batch index)


def schedule_1f1b(S: int, s: int, M: int) -> List[Op]:
    if S < 1 or not (0 <= s < S) or M < 1:
        raise ValueError("need S >= 1, 0 <= s < S, M >= 1")
    w = min(S - s - 1, M)
    ops: List[Op] = [("F", m) for m in range(w)]
    for i in range(M - w):
        ops.append(("F", w + i))
        ops.append(("B", i))
    ops.extend(("B", m) for m in range(M - w, M))
    return ops


def schedule_spec_reading(S: int, s: int, M: int) -> List[Op]:
    """SPEC S:L577 literally: warm-up min(S - s, M) forwards, then (B, F) pairs,
    then the remaining backwards.  Kept only to show the two readings agree."""
    w = min(S - s, M)
    ops: List[Op] = [("F", m) for m in range(w)]
    nf, nb = w, 0
    while nf < M:
        ops.append(("B", nb)); nb += 1
        ops.append(("F", nf)); nf += 1
    while nb < M:
        ops.append(("B", nb)); nb += 1
    return ops
