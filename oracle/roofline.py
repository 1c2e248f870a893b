"""O8 — comm-only 1F1B step roofline T* from the O2 event model.  TEST INFRASTRUCTURE ONLY.

T* is O2 with zero stage compute and message time bytes / link bandwidth
(900 GB/s per direction per GPU for NVLink 5, R4), in the "shared" link
model (per-GPU egress/ingress shared max-min) and, as the optimistic bound, the
"independent" model.  Pinned (tests/test_oracle_schedule_events.py::test_o8_step_roofline_pins)
by the hand-derived makespans: PP2 (M+1)*t and PP3 M3 8t shared / 6t independent.  As a
model of the hardware it is only validated against measured steps (8-GPU projections,
tests/test_projection_8gpu.py), not pinned.
"""
from __future__ import annotations

from .events import LinkModel, gbps_to_bytes_per_us, simulate

NVLINK_GBPS = 900.0


def step_roofline_us(S: int, M: int, msg_bytes: int, gbps: float = NVLINK_GBPS,
                     mode: str = "shared", K: int = 2) -> float:
    link = LinkModel(bw=gbps_to_bytes_per_us(gbps), mode=mode)
    return simulate(S, M, 0.0, 0.0, msg_bytes, msg_bytes, link, K=K).makespan


def tokens_per_s(M: int, seq: int, step_us: float, pipelines: int = 1) -> float:
    return pipelines * M * seq / (step_us * 1e-6)
