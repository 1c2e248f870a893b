"""NEXT-3 partition planner (paper_2602_18007_b200/partition.py), CPU only.

Pins: SPEC worked examples (S:L556 symmetric 32 layers -> 16-16; S:L557 per-layer ratio
1.133 -> 15-17 with fewer layers on the slower stage), the paper's ordering property
AMD < AMD+NVIDIA < NVIDIA under a proper partition and its converse under an inverted one
(P:L202-206), and the oracle's event model (oracle/events.py, O2) as an independent
simulator of every split (same argmin, same times)."""
import pytest

from oracle.events import LinkModel, simulate
from paper_2602_18007_b200.partition import iteration_time, optimize_partition


def test_spec_symmetric_split():
    assert optimize_partition(32, [1.0, 1.0], [2.0, 2.0], M=8) == [16, 16]


def test_spec_ratio_split():
    # stage 0 ("AMD") per-layer time 1.133x stage 1 ("NVIDIA")
    assert optimize_partition(32, [1.133, 1.0], [2 * 1.133, 2.0], M=8) == [15, 17]


def test_infeasible():
    with pytest.raises(ValueError):
        optimize_partition(1, [1.0, 1.0], [2.0, 2.0], M=4)


@pytest.mark.parametrize("comm", [0.0, 0.7])
def test_matches_oracle_event_model(comm):
    tf, tb, M, L = [1.3, 1.0], [2.5, 2.1], 6, 12
    for split in ([l, L - l] for l in range(1, L)):
        f = lambda s, m: split[s] * tf[s]
        b = lambda s, m: split[s] * tb[s]
        ref = simulate(2, M, f, b, 0, 0, LinkModel(bw=1.0, latency=comm), K=M + 1).makespan
        assert iteration_time(split, tf, tb, M, comm) == pytest.approx(ref, rel=1e-12)


def test_ordering_property():
    t_amd, t_nv, M, L = 1.133, 1.0, 8, 32
    amd = iteration_time([16, 16], [t_amd] * 2, [2 * t_amd] * 2, M)
    nv = iteration_time([16, 16], [t_nv] * 2, [2 * t_nv] * 2, M)
    het_split = optimize_partition(L, [t_amd, t_nv], [2 * t_amd, 2 * t_nv], M)
    het = iteration_time(het_split, [t_amd, t_nv], [2 * t_amd, 2 * t_nv], M)
    assert nv < het < amd                                   # P:L204 AMD < AMD+NVIDIA < NVIDIA
    inverted = iteration_time([het_split[1], het_split[0]], [t_amd, t_nv], [2 * t_amd, 2 * t_nv], M)
    assert inverted > amd > het        # improper partitioning underperforms even AMD-homo
