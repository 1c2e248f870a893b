"""O7 — fp32 -> bf16 round-to-nearest-even and bf16 -> fp32 widening.  TEST INFRASTRUCTURE ONLY.

Used for the bf16 boundary variant of the toy pipeline (BJ north_star: "within
1e-3 relative error (bf16) on the toy-model loss").  Definition (IEEE-754
round-to-nearest-even applied to the top 16 bits of the fp32 encoding u):
    b = (u + 0x7FFF + ((u >> 16) & 1)) >> 16          for non-NaN u
NaN inputs map to the quiet NaN 0x7FC0 with the sign kept (a NaN class, R8).

Pinned by tests/test_oracle_bf16.py against the library special case torch CPU
`.to(torch.bfloat16)` on random and edge-case inputs (ties, subnormals, Inf, max).
"""
from __future__ import annotations

import numpy as np


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    if nan.any():
        sign = ((u >> 16) & 0x8000).astype(np.uint16)
        rounded = np.where(nan, sign | np.uint16(0x7FC0), rounded)
    return rounded


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def round_through_bf16(x: np.ndarray) -> np.ndarray:
    """x (any float dtype) -> fp32 (numpy RNE) -> bf16 RNE -> widened back to x's dtype."""
    dt = np.asarray(x).dtype
    return bf16_bits_to_f32(f32_to_bf16_bits(np.asarray(x, dtype=np.float32))).astype(dt)
