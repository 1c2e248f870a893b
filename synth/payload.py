"""Synthetic stage-boundary payloads: a counter-based SplitMix64 stream per message.

Recipe:

    mix(z):  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
             z = (z ^ (z >> 27)) * 0x94D049BB133111EB
             return z ^ (z >> 31)                        (all mod 2**64)
    GAMMA = 0x9E3779B97F4A7C15
    key   = seed<<48 ^ step<<32 ^ boundary<<24 ^ dir<<23 ^ mb
    base  = mix(key + GAMMA)          (= first output of SplitMix64 seeded with key)
    word[w] = mix(base + (w+1)*GAMMA) (= SplitMix64 stream seeded with base)

The payload is the little-endian u64 word array truncated to `nbytes`.  Every
16-bit pattern (including bf16 NaN/Inf/subnormal encodings) occurs, so any
accidental float conversion on the transfer path changes the bytes.

Named sources:
  * activation source X_m of stage 0  : payload_bytes(seed, step, SRC_BOUNDARY, 0, m)
  * loss gradient     G_m of stage S-1: payload_bytes(seed, step, SRC_BOUNDARY, 1, m)
  * XOR-proxy masks   H_F(s,m)/H_B(s,m): payload_bytes(seed ^ MASK_TAG, step, s, 0|1, m)
  * raw message for (boundary b, dir d, mb m): payload_bytes(seed, step, b, d, m)

The device fill kernel (`ppc_fill_splitmix`) implements the same generator
independently in CUDA; tests compare it against this module.
"""
from __future__ import annotations

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
M1 = 0xBF58476D1CE4E5B9
M2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1

SRC_BOUNDARY = 0xFF      # boundary field used for stage-0 activations / last-stage gradients
MASK_TAG = 0x8000        # seed tag for the XOR stage-proxy masks (seed < 2**15)


def make_key(seed: int, step: int, boundary: int, direction: int, mb: int) -> int:
    if not (0 <= seed < 1 << 16 and 0 <= step < 1 << 16):
        raise ValueError("seed and step must be < 2**16")
    if not (0 <= boundary < 1 << 8 and direction in (0, 1) and 0 <= mb < 1 << 23):
        raise ValueError("boundary < 2**8, dir in {0,1}, mb < 2**23")
    return (seed << 48) ^ (step << 32) ^ (boundary << 24) ^ (direction << 23) ^ mb


def mix_scalar(z: int) -> int:
    z &= MASK64
    z = ((z ^ (z >> 30)) * M1) & MASK64
    z = ((z ^ (z >> 27)) * M2) & MASK64
    return z ^ (z >> 31)


def _mix_vec(z: np.ndarray) -> np.ndarray:
    z = z.copy()
    z ^= z >> np.uint64(30)
    z *= np.uint64(M1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(M2)
    z ^= z >> np.uint64(31)
    return z


def splitmix64_stream(state: int, n: int) -> np.ndarray:
    """n outputs of the textbook SplitMix64 generator seeded with `state`
    (x += GAMMA; return mix(x)), as uint64."""
    w = np.arange(1, n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(state & MASK64) + w * np.uint64(GAMMA)
        return _mix_vec(z)


def payload_words(seed: int, step: int, boundary: int, direction: int, mb: int, nwords: int) -> np.ndarray:
    key = make_key(seed, step, boundary, direction, mb)
    base = mix_scalar(key + GAMMA)
    return splitmix64_stream(base, nwords)


def payload_bytes(seed: int, step: int, boundary: int, direction: int, mb: int, nbytes: int) -> np.ndarray:
    """uint8 array of `nbytes` payload bytes (little-endian words, truncated)."""
    nwords = (nbytes + 7) // 8
    w = payload_words(seed, step, boundary, direction, mb, nwords)
    return w.astype("<u8", copy=False).view(np.uint8)[:nbytes].copy()


def source_activation(seed: int, step: int, mb: int, nbytes: int) -> np.ndarray:
    return payload_bytes(seed, step, SRC_BOUNDARY, 0, mb, nbytes)


def source_gradient(seed: int, step: int, mb: int, nbytes: int) -> np.ndarray:
    return payload_bytes(seed, step, SRC_BOUNDARY, 1, mb, nbytes)


def proxy_mask(seed: int, step: int, stage: int, direction: int, mb: int, nbytes: int) -> np.ndarray:
    return payload_bytes(seed ^ MASK_TAG, step, stage, direction, mb, nbytes)
