"""Pins for oracle/collectives.py (NEXT-2): SPEC worked examples and composition == plain sum."""
import numpy as np
import pytest

from oracle.collectives import allreduce_reference, composed_allreduce


def test_spec_rank_id_allreduce():
    vals = {r: np.array([float(r)]) for r in range(4)}
    assert allreduce_reference(vals, [0, 1, 2, 3])[0] == 6.0


def test_spec_hetero_example():
    # subgroups {1,2 | 3,4}: ranks 0,1 on stage 0 and 2,3 on stage 1 (pp=2, dp=2)
    vals = {0: np.array([1.0]), 1: np.array([2.0]), 2: np.array([3.0]), 3: np.array([4.0])}
    out = composed_allreduce(vals, 4, tp=1, pp=2, dp=2)
    assert all(out[r][0] == 10.0 for r in range(4))


@pytest.mark.parametrize("tp,pp,dp", [(1, 2, 2), (1, 4, 1), (2, 2, 2), (1, 3, 2)])
def test_composition_equals_plain_sum(tp, pp, dp):
    world = tp * pp * dp
    rng = np.random.default_rng(0)
    vals = {r: rng.integers(-1000, 1000, 37).astype(np.float64) for r in range(world)}
    out = composed_allreduce(vals, world, tp, pp, dp)
    for r in range(world):
        group = [q for q in range(world) if q % tp == r % tp]
        assert np.array_equal(out[r], allreduce_reference(vals, group))


def test_tp_gather_reference_is_the_inverse_of_slicing():
    from oracle.collectives import tp_gather_reference
    full = np.arange(1001, dtype=np.uint8)
    for tp in (1, 2, 7):
        n = len(full) // tp * tp
        parts = [full[i * (n // tp):(i + 1) * (n // tp)] for i in range(tp)]
        assert np.array_equal(tp_gather_reference(parts), full[:n])
