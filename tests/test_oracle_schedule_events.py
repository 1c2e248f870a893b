"""Pins for oracle O1 (schedule) and O2 (event model).  CPU only.

Pins used (none re-types the oracle's own formula):
  * brute force: every in-flight-bounded per-stage order is simulated; 1F1B must be
    the unique makespan argmin under uniform costs (SURVEY App. A2 finding);
  * closed forms: zero-comm makespan (M+S-1)(f+b); PP2 comm-only (M+1)*t_msg
    (critical path derived by hand in DESIGN.md R5); SPEC 1-stage case M(f+b);
  * SPEC worked examples (tests/golden/spec_examples.txt);
  * invariants: deadlock-free for K >= 1, occupancy <= min(S-s, M), trace validity.
"""
import itertools
import os
import random

import pytest

from oracle.events import (Deadlock, LinkModel, gbps_to_bytes_per_us, pipelined_time,
                           simulate, validate_trace, wire_time)
from oracle.schedule import schedule_1f1b, schedule_spec_reading

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _enumerate_orders(s, S, M):
    """All per-stage orders: F ascending, B ascending, F_m before B_m, at most
    min(S - s, M) micro-batches in flight (SURVEY App. A3 bound)."""
    cap = min(S - s, M)
    out = []

    def rec(nf, nb, cur):
        if nf == M and nb == M:
            out.append(list(cur))
            return
        if nf < M and nf - nb < cap:
            cur.append(("F", nf)); rec(nf + 1, nb, cur); cur.pop()
        if nb < nf:
            cur.append(("B", nb)); rec(nf, nb + 1, cur); cur.pop()
    rec(0, 0, [])
    return out


def test_schedule_counts_and_order():
    for S in range(1, 9):
        for s in range(S):
            for M in range(1, 20):
                ops = schedule_1f1b(S, s, M)
                assert len(ops) == 2 * M
                fs = [m for k, m in ops if k == "F"]
                bs = [m for k, m in ops if k == "B"]
                assert fs == list(range(M)) and bs == list(range(M))
                # F_m precedes B_m; in flight never exceeds min(S - s, M)
                done_f, done_b = 0, 0
                for k, m in ops:
                    if k == "F":
                        done_f += 1
                    else:
                        assert m < done_f
                        done_b += 1
                    assert done_f - done_b <= min(S - s, M)


def test_spec_warmup_reading_is_identical():
    # S:L577 writes warmup = min(pp - s, M) with (B, F) steady pairs (R2)
    for S in range(1, 9):
        for s in range(S):
            for M in range(1, 40):
                assert schedule_1f1b(S, s, M) == schedule_spec_reading(S, s, M)


def test_invalid_args():
    for bad in [(0, 0, 1), (2, 2, 1), (2, -1, 1), (2, 0, 0)]:
        with pytest.raises(ValueError):
            schedule_1f1b(*bad)


@pytest.mark.parametrize("S,M", [(2, 2), (2, 3), (2, 4), (3, 2), (3, 3), (3, 4), (4, 3), (4, 4)])
@pytest.mark.parametrize("f,b,c", [(1, 1, 0), (1, 2, 0), (1, 2, 0.5), (2, 3, 1)])
def test_brute_force_1f1b_unique_argmin(S, M, f, b, c):
    per = [_enumerate_orders(s, S, M) for s in range(S)]
    best, argmins = None, []
    for combo in itertools.product(*per):
        try:
            r = simulate(S, M, f, b, 0, 0, LinkModel(bw=1.0, latency=c), K=M + 1,
                         orders=[list(x) for x in combo])
        except Deadlock:
            continue
        if best is None or r.makespan < best - 1e-9:
            best, argmins = r.makespan, [combo]
        elif abs(r.makespan - best) < 1e-9:
            argmins.append(combo)
    ref = [schedule_1f1b(S, s, M) for s in range(S)]
    assert len(argmins) == 1 and [list(x) for x in argmins[0]] == ref
    if c == 0:
        assert best == (M + S - 1) * (f + b)


@pytest.mark.parametrize("S,M,f,b", [(1, 5, 1.0, 2.0), (2, 8, 3.0, 5.0), (4, 16, 1.0, 2.0),
                                     (8, 32, 2.0, 3.0), (5, 3, 1.0, 1.0)])
def test_zero_comm_closed_form(S, M, f, b):
    r = simulate(S, M, f, b, 0, 0, LinkModel(bw=1.0), K=2)
    validate_trace(r, S)
    assert r.makespan == pytest.approx((M + S - 1) * (f + b), abs=1e-9)


def test_spec_one_stage_case():
    # 1 stage, m micro-batches, L layers of time t -> m * L * (t_fwd + t_bwd)
    L, tf, tb, m = 16, 0.7, 1.3, 6
    r = simulate(1, m, L * tf, L * tb, 0, 0, LinkModel(bw=1.0))
    assert r.makespan == pytest.approx(m * L * (tf + tb))


@pytest.mark.parametrize("M", [1, 2, 8, 16])
@pytest.mark.parametrize("mode", ["independent", "shared"])
def test_pp2_comm_only_closed_form(M, mode):
    # Hand-derived (R5): with zero compute the critical path alternates one
    # FWD and one BWD message per micro-batch after the first: T = (M + 1) * t_msg.
    nbytes = 32 << 20
    bw = gbps_to_bytes_per_us(900)
    r = simulate(2, M, 0.0, 0.0, nbytes, nbytes, LinkModel(bw=bw, mode=mode), K=2)
    assert r.makespan == pytest.approx((M + 1) * nbytes / bw, rel=1e-12)


def _golden_examples():
    rows = {}
    with open(os.path.join(GOLDEN, "spec_examples.txt")) as fh:
        for line in fh:
            line = line.split("#")[0].strip()
            if not line:
                continue
            name, cite, inputs, expected, tol = [x.strip() for x in line.split("|")]
            rows[name] = (float(expected), float(tol))
    return rows


def test_spec_worked_examples():
    g = _golden_examples()
    gb = gbps_to_bytes_per_us
    cases = {
        "wire_time_nic": wire_time(gb(100), 5.0, 1 << 30),
        "wire_time_nvlink": wire_time(gb(900), 1.0, 1 << 30),
        "dev_copy_fast": wire_time(gb(3000), 0.0, 1 << 30),
        "dev_copy_slow": wire_time(gb(64), 0.0, 1 << 30),
        "net_4mib": wire_time(gb(100), 5.0, 4 << 20),
        "pipelined_time": pipelined_time([2, 5, 2], 10),
    }
    for name, got in cases.items():
        exp, tol = g[name]
        assert abs(got - exp) <= tol, (name, got, exp)
    assert wire_time(gb(900), 3.0, 0) == 3.0                 # 0 bytes -> latency only
    assert pipelined_time([2, 5, 2], 1) == 9                  # 1 chunk -> sum
    assert pipelined_time([3, 3, 3], 7) == 3 * (3 + 7 - 1)    # symmetric case
    with pytest.raises(ValueError):
        pipelined_time([1], 0)


def test_deadlock_free_random():
    # blocking sends into K-slot rings never deadlock for K >= 1
    rng = random.Random(1234)
    for trial in range(250):
        S = rng.randint(1, 6)
        M = rng.randint(1, 10)
        K = rng.choice([1, 2, 3])
        fc = {(s, m): rng.uniform(0.1, 3) for s in range(S) for m in range(M)}
        bc = {(s, m): rng.uniform(0.1, 5) for s in range(S) for m in range(M)}
        link = LinkModel(bw=rng.uniform(0.5, 4), latency=rng.uniform(0, 1),
                         mode=rng.choice(["independent", "shared"]))
        nb = rng.randint(0, 8)
        r = simulate(S, M, lambda s, m: fc[s, m], lambda s, m: bc[s, m], nb, nb, link, K=K,
                     copy_out=rng.choice([0.0, 0.2]), blocking_sends=rng.random() < 0.5)
        validate_trace(r, S)
        assert len(r.ops) == 2 * S * M
        assert len(r.msgs) == 2 * (S - 1) * M


def test_occupancy_bound():
    # unconsumed FWD messages at boundary s <= min(S - s, M)
    rng = random.Random(7)
    attained = False
    for trial in range(200):
        S = rng.randint(2, 7)
        M = rng.randint(1, 12)
        fc = {(s, m): rng.uniform(0.01, 3) for s in range(S) for m in range(M)}
        bc = {(s, m): rng.uniform(0.01, 3) for s in range(S) for m in range(M)}
        r = simulate(S, M, lambda s, m: fc[s, m], lambda s, m: bc[s, m], 1, 1,
                     LinkModel(bw=rng.uniform(0.2, 20)), K=M + 1)
        for (d, bnd), occ in r.max_occupancy.items():
            if d == 0:
                assert occ <= min(S - bnd, M)
                attained |= occ == min(S - bnd, M) and S - bnd > 1
    assert attained


def test_shared_never_faster_than_independent():
    for S, M in [(2, 4), (3, 6), (4, 8)]:
        nb = 1 << 20
        a = simulate(S, M, 0.5, 1.0, nb, nb, LinkModel(bw=1e5, mode="independent")).makespan
        c = simulate(S, M, 0.5, 1.0, nb, nb, LinkModel(bw=1e5, mode="shared")).makespan
        assert c >= a - 1e-9


def test_trace_csv_schema_and_order():
    r = simulate(3, 4, 1.0, 2.0, 100, 100, LinkModel(bw=10.0, latency=0.5))
    csv = r.trace_csv().splitlines()
    assert csv[0] == "t_start_us,t_end_us,src,dst,path,size_bytes,segment_kind"
    rows = r.trace_rows()
    assert len(rows) == 2 * 2 * 4
    keys = [(row[0], row[2]) for row in rows]
    assert keys == sorted(keys)


# ---- max-min sharing of per-GPU egress / ingress (O2 "shared"; R6).
# Hand-derived progressive-filling results; a filling that ignores the ingress constraint,
# never releases capacity, or releases it from the wrong resource fails at least one.
def _rates(flows, egress=1.0, ingress=1.0):
    from oracle.events import Msg, _maxmin_rates
    ms = [Msg(0, 0, a, b, i + 1, 0, 1, 0.0) for i, (a, b) in enumerate(flows)]
    _maxmin_rates(ms, LinkModel(bw=1.0, mode="shared", egress=egress, ingress=ingress))
    return [m.rate for m in ms]


def test_maxmin_two_flows_share_one_egress():
    # A->B, A->C: GPU A's egress (1) is the only shared resource -> 1/2 each
    assert _rates([(0, 1), (0, 2)]) == pytest.approx([0.5, 0.5])


def test_maxmin_ingress_binds():
    # A->C, B->C share C's ingress -> 1/2 each; D->E alone -> 1 (an egress-only model
    # would give all three 1)
    assert _rates([(0, 2), (1, 2), (3, 4)]) == pytest.approx([0.5, 0.5, 1.0])


def test_maxmin_three_flow_classic():
    # A->B, A->C, D->C: A's egress and C's ingress both have 2 users (share 1/2); after
    # freezing A's flows at 1/2, C's ingress has 1/2 left for D->C -> 1/2, 1/2, 1/2
    assert _rates([(0, 1), (0, 2), (3, 2)]) == pytest.approx([0.5, 0.5, 0.5])


def test_maxmin_capacity_released_from_the_right_resource():
    # A->B, A->C, A->D, E->D: A's egress (3 users, 1/3) is tightest; D's ingress keeps
    # 1 - 1/3 = 2/3 for E->D (not 1/2: the freed share must be subtracted from D's ingress)
    assert _rates([(0, 1), (0, 2), (0, 3), (4, 3)]) == pytest.approx([1 / 3] * 3 + [2 / 3])


def test_maxmin_unequal_caps():
    # egress 1, ingress 0.6: a lone flow gets min(1, 0.6); two flows into one GPU 0.3 each
    assert _rates([(0, 1)], ingress=0.6) == pytest.approx([0.6])
    assert _rates([(0, 1), (2, 1)], ingress=0.6) == pytest.approx([0.3, 0.3])


@pytest.mark.parametrize("mode,units", [("shared", 8), ("independent", 6)])
def test_pp3_comm_only_makespan_hand_derived(mode, units):
    """PP3, M = 3, zero compute, message time t (DESIGN.md §2 R6, worked out there step by
    step): the middle stage's FWD (c2) and BWD (e0) sends overlap in [4t, 6t) and share its
    egress, and stage 1's ingress is shared by a2 and d0 in [2t, 4t) -> T = 8t; with
    independent links the same schedule takes 6t."""
    nbytes, bw = 1 << 20, 1e5
    r = simulate(3, 3, 0.0, 0.0, nbytes, nbytes, LinkModel(bw=bw, mode=mode), K=4)
    validate_trace(r, 3)
    assert r.makespan == pytest.approx(units * nbytes / bw, rel=1e-12)


def test_o8_step_roofline_pins():
    """O8 (oracle/roofline.py): the comm-only T* equals the hand-derived makespans — PP2
    (M+1)·t (R5) and PP3 M3 8t shared / 6t independent (§2a) — at 900 GB/s, and
    tokens/s is M·seq / T (C2: 335.544 µs -> 97.66 M tok/s)."""
    from oracle.roofline import step_roofline_us, tokens_per_s
    nb = 32 << 20
    t = nb / gbps_to_bytes_per_us(900)                       # 37.28 us
    assert step_roofline_us(2, 8, nb) == pytest.approx(9 * t, rel=1e-12)
    assert step_roofline_us(2, 8, nb) == pytest.approx(335.54432, abs=1e-5)
    assert step_roofline_us(3, 3, nb, K=4) == pytest.approx(8 * t, rel=1e-12)
    assert step_roofline_us(3, 3, nb, mode="independent", K=4) == pytest.approx(6 * t, rel=1e-12)
    assert tokens_per_s(8, 4096, 335.54432) == pytest.approx(97.66e6, rel=1e-3)
    assert tokens_per_s(8, 4096, 500.0, pipelines=2) == pytest.approx(2 * 8 * 4096 / 500e-6)
