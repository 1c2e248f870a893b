"""O2 — discrete-event timing model of one 1F1B step.  TEST INFRASTRUCTURE ONLY.

Follows SPEC.md:
  * wire_time = latency + size / bandwidth
  * pipelined_time = sum(stage_times) + (n - 1) * max(stage_times)
  * ScheduleTrace: per-stage events, dependency-correct, iteration time = max t_end
                                                                          
  * trace CSV columns t_start_us,t_end_us,src,dst,path,size_bytes,segment_kind,
    ordered by (t_start, src_rank, seq)
and the dependency structure of a non-interleaved pipeline (R2/R5):
  * F_m at stage s needs the FWD message m from stage s-1 delivered (s > 0);
  * B_m at stage s needs the BWD message m from stage s+1 delivered (s < S-1);
    at s = S-1, F_m precedes B_m in the stage's own op order;
  * after F_m (s < S-1) the stage sends FWD m to s+1; after B_m (s > 0) it sends BWD m
    to s-1.  Sends are asynchronous (a separate stream in the GPU design) unless
    `blocking_sends`, in which case the stage waits until the message has a slot;
  * each (src, dst) link carries its messages FIFO, in send order;
  * a message may start only when its ring slot is free: with K slots, message seq
    needs message seq-K consumed (credit protocol);
  * a message is consumed when the receiving op starts its copy-out; the slot frees
    `copy_out` microseconds later.

Link models (R6):
  * "independent": every link runs at `bw` on its own (optimistic bound);
  * "shared": links active at the same time share each GPU's egress and ingress
    capacity max-min fairly (NVSwitch caps per GPU, not per pair).
A message spends `latency` before its bytes start to flow, then bytes / rate.

Pinned by tests/test_oracle_events.py: SPEC worked examples (wire_time,
pipelined_time), the zero-comm closed form (M+S-1)(f+b), SPEC's 1-stage case,
deadlock freedom for K >= 1 on random costs, the occupancy bound min(S-s, M), and
trace validity (no per-stage overlap; every recv after its send).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple, Union

from .schedule import schedule_1f1b

EPS = 1e-9
FWD, BWD = 0, 1


def wire_time(bandwidth_bytes_per_us: float, latency_us: float, size_bytes: int) -> float:
    """latency + size / bandwidth (double precision)."""
    if size_bytes < 0:
        raise ValueError("size must be >= 0")
    return latency_us + size_bytes / bandwidth_bytes_per_us


def pipelined_time(stage_times: Sequence[float], num_chunks: int) -> float:
    """sum(stage_times) + (num_chunks - 1) * max(stage_times)."""
    if num_chunks < 1 or any(t < 0 for t in stage_times):
        raise ValueError("num_chunks >= 1 and stage times >= 0")
    return sum(stage_times) + (num_chunks - 1) * max(stage_times)


def gbps_to_bytes_per_us(gbps: float) -> float:
    return gbps * 1e9 / 1e6


class Deadlock(RuntimeError):
    pass


@dataclass
class LinkModel:
    bw: float                      # bytes per microsecond per link (900 GB/s -> 9e5)
    latency: float = 0.0           # microseconds before a message's bytes flow
    mode: str = "independent"      # "independent" | "shared"
    egress: Optional[float] = None  # per-GPU egress cap (shared mode), default bw
    ingress: Optional[float] = None


@dataclass
class Msg:
    direction: int
    boundary: int       # boundary b joins stages b and b+1
    src: int
    dst: int
    seq: int            # 1-based per (boundary, direction)
    mb: int
    nbytes: int
    t_ready: float
    t_start: Optional[float] = None
    t_flow: Optional[float] = None     # latency over, bytes start flowing
    t_end: Optional[float] = None      # delivered
    t_consumed: Optional[float] = None  # receiver started copy-out
    t_free: Optional[float] = None      # slot free again
    remaining: float = 0.0
    rate: float = 0.0


@dataclass
class SimResult:
    makespan: float
    ops: List[dict]
    msgs: List[Msg]
    max_occupancy: Dict[Tuple[int, int], int] = field(default_factory=dict)

    def trace_rows(self) -> List[tuple]:
        """SPEC S:L262 CSV rows ordered by (t_start, src_rank, seq)."""
        rows = []
        for m in self.msgs:
            rows.append((m.t_start, m.t_end, m.src, m.dst, "device_direct", m.nbytes,
                         "fwd" if m.direction == FWD else "bwd", m.seq))
        rows.sort(key=lambda r: (r[0], r[2], r[7]))
        return [r[:7] for r in rows]

    def trace_csv(self) -> str:
        out = ["t_start_us,t_end_us,src,dst,path,size_bytes,segment_kind"]
        for r in self.trace_rows():
            out.append(f"{r[0]:.6f},{r[1]:.6f},{r[2]},{r[3]},{r[4]},{r[5]},{r[6]}")
        return "\n".join(out) + "\n"


Cost = Union[float, Callable[[int, int], float]]


def _cost(c: Cost, s: int, m: int) -> float:
    return float(c(s, m)) if callable(c) else float(c)


def _maxmin_rates(active: List[Msg], link: LinkModel) -> None:
    if link.mode == "independent":
        for m in active:
            m.rate = link.bw
        return
    if link.mode != "shared":
        raise ValueError(link.mode)
    eg = link.egress if link.egress is not None else link.bw
    ing = link.ingress if link.ingress is not None else link.bw
    cap: Dict[tuple, float] = {}
    users: Dict[tuple, List[Msg]] = {}
    for m in active:
        for r, c in ((("out", m.src), eg), (("in", m.dst), ing)):
            cap.setdefault(r, c)
            users.setdefault(r, []).append(m)
    frozen = set()
    # progressive filling: repeatedly saturate the tightest resource
    while len(frozen) < len(active):
        best_r, best_share = None, math.inf
        for r, us in users.items():
            n = sum(1 for m in us if id(m) not in frozen)
            if n == 0:
                continue
            share = cap[r] / n
            if share < best_share - EPS:
                best_r, best_share = r, share
        for m in users[best_r]:
            if id(m) in frozen:
                continue
            m.rate = best_share
            frozen.add(id(m))
            for r in (("out", m.src), ("in", m.dst)):
                cap[r] -= best_share
    return


def simulate(S: int, M: int, f: Cost, b: Cost, fwd_bytes: int, bwd_bytes: int,
             link: LinkModel, K: int = 2, orders: Optional[List[List[tuple]]] = None,
             copy_out: float = 0.0, blocking_sends: bool = False) -> SimResult:
    """Simulate one step of a pipeline of S stages over M micro-batches.

    `orders[s]` overrides the per-stage op order (default: O1's 1F1B).  Times in us.
    """
    if K < 1:
        raise ValueError("K >= 1")
    orders = orders or [schedule_1f1b(S, s, M) for s in range(S)]
    idx = [0] * S
    busy_until = [0.0] * S
    running: List[Optional[tuple]] = [None] * S   # (kind, m, t_start, t_end)
    blocked_on: List[Optional[Msg]] = [None] * S  # blocking send waiting for a slot
    ops_out: List[dict] = []
    fifo: Dict[Tuple[int, int], List[Msg]] = {}
    msgs: Dict[Tuple[int, int, int], Msg] = {}    # (direction, boundary, mb) -> msg
    chan_msgs: Dict[Tuple[int, int], Dict[int, Msg]] = {}  # (dir, boundary) -> seq -> msg
    sent_count: Dict[Tuple[int, int], int] = {}
    occ: Dict[Tuple[int, int], int] = {}
    max_occ: Dict[Tuple[int, int], int] = {}
    t = 0.0

    def make_msg(direction: int, s: int, m: int, now: float) -> Msg:
        if direction == FWD:
            boundary, src, dst, nb = s, s, s + 1, fwd_bytes
        else:
            boundary, src, dst, nb = s - 1, s, s - 1, bwd_bytes
        ch = (direction, boundary)
        seq = sent_count.get(ch, 0) + 1
        sent_count[ch] = seq
        msg = Msg(direction, boundary, src, dst, seq, m, nb, now, remaining=float(nb))
        msgs[(direction, boundary, m)] = msg
        chan_msgs.setdefault(ch, {})[seq] = msg
        fifo.setdefault((src, dst), []).append(msg)
        return msg

    def slot_free(msg: Msg, now: float) -> bool:
        if msg.seq <= K:
            return True
        prev = chan_msgs[(msg.direction, msg.boundary)].get(msg.seq - K)
        return prev is not None and prev.t_free is not None and prev.t_free <= now + EPS

    total_ops = sum(len(o) for o in orders)
    done_ops = 0
    while True:
        # ---- zero-time progress at time t ----
        progress = True
        while progress:
            progress = False
            # finish ops ending at t
            for s in range(S):
                r = running[s]
                if r is not None and r[3] <= t + EPS:
                    kind, m, ts, te = r
                    ops_out.append(dict(stage=s, kind=kind, mb=m, t_start=ts, t_end=te))
                    running[s] = None
                    done_ops += 1
                    progress = True
                    if kind == "F" and s < S - 1:
                        msg = make_msg(FWD, s, m, te)
                    elif kind == "B" and s > 0:
                        msg = make_msg(BWD, s, m, te)
                    else:
                        msg = None
                    if msg is not None and blocking_sends:
                        blocked_on[s] = msg
            # deliver messages whose bytes have all flowed
            for q in fifo.values():
                while q and q[0].t_start is not None and q[0].t_end is None \
                        and q[0].t_flow <= t + EPS and q[0].remaining <= EPS * max(1.0, q[0].nbytes):
                    q[0].t_end = t
                    q[0].remaining = 0.0
                    q.pop(0)
                    progress = True
            # start link transfers
            for (src, dst), q in fifo.items():
                if not q:
                    continue
                head = q[0]
                if head.t_start is not None:
                    continue
                if not slot_free(head, t):
                    continue
                head.t_start = t
                head.t_flow = t + link.latency
                ch = (head.direction, head.boundary)
                occ[ch] = occ.get(ch, 0) + 1
                max_occ[ch] = max(max_occ.get(ch, 0), occ[ch])
                progress = True
            # release blocked senders whose message started
            for s in range(S):
                if blocked_on[s] is not None and blocked_on[s].t_start is not None:
                    blocked_on[s] = None
                    progress = True
            # start ops
            for s in range(S):
                if running[s] is not None or blocked_on[s] is not None or idx[s] >= len(orders[s]):
                    continue
                kind, m = orders[s][idx[s]]
                dep = None
                if kind == "F" and s > 0:
                    dep = msgs.get((FWD, s - 1, m))
                    need = True
                elif kind == "B" and s < S - 1:
                    dep = msgs.get((BWD, s, m))
                    need = True
                else:
                    need = False
                if need and (dep is None or dep.t_end is None or dep.t_end > t + EPS):
                    continue
                dur = (copy_out if need else 0.0) + _cost(f if kind == "F" else b, s, m)
                if need:
                    dep.t_consumed = t
                    dep.t_free = t + copy_out
                    ch = (dep.direction, dep.boundary)
                    occ[ch] -= 1
                running[s] = (kind, m, t, t + dur)
                idx[s] += 1
                progress = True
                if dur <= EPS:
                    running[s] = (kind, m, t, t)
        if done_ops == total_ops and all(not q or q[-1].t_end is not None for q in fifo.values()):
            break
        # ---- next event ----
        flowing = [m for q in fifo.values() for m in q[:1]
                   if m.t_start is not None and m.t_end is None and m.t_flow <= t + EPS]
        _maxmin_rates(flowing, link)
        cands = []
        for s in range(S):
            if running[s] is not None:
                cands.append(running[s][3])
        for q in fifo.values():
            if q and q[0].t_start is not None and q[0].t_end is None:
                h = q[0]
                if h.t_flow > t + EPS:
                    cands.append(h.t_flow)
                elif h.rate > 0:
                    cands.append(t + h.remaining / h.rate)
        for chm in chan_msgs.values():
            for msg in chm.values():
                if msg.t_free is not None and msg.t_free > t + EPS:
                    cands.append(msg.t_free)
        cands = [c for c in cands if c > t + EPS]
        if not cands:
            raise Deadlock(f"no progress at t={t}: idx={idx} of {[len(o) for o in orders]}")
        tn = min(cands)
        dt = tn - t
        for m in flowing:
            m.remaining -= m.rate * dt
        t = tn
    # rebuild: delivered messages were popped from FIFOs; collect from msgs map
    all_msgs = sorted(msgs.values(), key=lambda x: (x.t_start, x.src, x.seq))
    makespan = max([o["t_end"] for o in ops_out] + [m.t_end for m in all_msgs] + [0.0])
    return SimResult(makespan, ops_out, all_msgs, max_occ)


def validate_trace(res: SimResult, S: int) -> None:
    """ScheduleTrace invariants: ops on one stage never overlap; every
    receiving op starts after its message was delivered; every message starts
    after the op that produced it ended."""
    by_stage: Dict[int, List[dict]] = {}
    for o in res.ops:
        by_stage.setdefault(o["stage"], []).append(o)
    for s, lst in by_stage.items():
        lst.sort(key=lambda o: (o["t_start"], o["t_end"]))
        for a, c in zip(lst, lst[1:]):
            if c["t_start"] < a["t_end"] - EPS:
                raise AssertionError(f"overlap on stage {s}: {a} {c}")
    op_at = {(o["stage"], o["kind"], o["mb"]): o for o in res.ops}
    for m in res.msgs:
        kind = "F" if m.direction == FWD else "B"
        prod = op_at[(m.src, kind, m.mb)]
        cons = op_at[(m.dst, kind, m.mb)]
        if m.t_start < prod["t_end"] - EPS:
            raise AssertionError(f"message {m} starts before its producer ends")
        if cons["t_start"] < m.t_end - EPS:
            raise AssertionError(f"consumer of {m} starts before delivery")
