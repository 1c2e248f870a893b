"""Pins for oracle O3 (byte transfer), O5 (XOR stage proxy run) and the payload inputs.

Pins: SplitMix64 textbook outputs (tests/golden/splitmix64.txt), identity of
delivered bytes (SPEC S:L264 data-plane integrity), exactly-once/in-order logs,
error cases forced by SPEC (S:L361 SizeMismatch) and the XOR closed form.
"""
import os
import random

import numpy as np
import pytest

from oracle.proxy import run_1f1b, xor_closed_form, xor_stage
from oracle.transfer import (BWD, FWD, MAGIC, Channel, OrderError, SizeMismatch, TransferError,
                             WouldBlock, digest, pack_header, unpack_header)
from synth import payload as P

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_textbook_vectors():
    with open(os.path.join(GOLDEN, "splitmix64.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            seed, outs = line.split(":")
            want = [int(x, 16) for x in outs.split()]
            got = [int(x) for x in P.splitmix64_stream(int(seed), len(want))]
            assert got == want


def test_payload_structure():
    # base = first SplitMix64 output seeded with the key; words = stream seeded with base
    key = P.make_key(42, 1, 2, 0, 7)
    base = int(P.splitmix64_stream(key, 1)[0])
    assert np.array_equal(P.payload_words(42, 1, 2, 0, 7, 5), P.splitmix64_stream(base, 5))
    b = P.payload_bytes(42, 0, 0, 0, 0, 13)
    w = P.payload_words(42, 0, 0, 0, 0, 2)
    assert b.tobytes() == w.astype("<u8").tobytes()[:13]
    # every bf16 bit pattern occurs in a 4 MiB payload (raw patterns, R12)
    u16 = P.payload_bytes(42, 0, 0, 0, 0, 4 << 20).view(np.uint16)
    assert np.unique(u16).size == 65536
    # distinct keys give independent streams
    a = P.payload_bytes(42, 0, 0, 0, 1, 64)
    c = P.payload_bytes(42, 0, 0, 1, 1, 64)
    assert not np.array_equal(a, c)
    with pytest.raises(ValueError):
        P.make_key(1 << 16, 0, 0, 0, 0)


def test_header_layout():
    h = pack_header(1, 3, 12345, 9, 4, 2)
    assert len(h) == 64
    assert h[:4] == b"CPCH"          # 0x48435043 little-endian
    d = unpack_header(h)
    assert d == dict(magic=MAGIC, dir=1, boundary=3, bytes=12345, seq=9, mb=4, step=2)


def test_identity_random_payloads():
    rng = np.random.default_rng(0)
    for K in (1, 2, 3):
        ch = Channel(FWD, 0, K, 1 << 20)
        for i in range(120):
            n = int(rng.integers(0, 1 << 20))
            data = rng.integers(0, 256, n, dtype=np.uint8)
            ch.send(data, mb=i)
            out = ch.recv(n, mb=i)
            assert out.tobytes() == data.tobytes()       # library special case: bytes copy
        assert [r[0] for r in ch.log] == list(range(1, 121))
        assert [r[1] for r in ch.log] == list(range(120))


def test_errors():
    ch = Channel(FWD, 0, 2, 1024)
    with pytest.raises(TransferError):
        ch.send(np.zeros(2048, np.uint8), 0)
    ch.send(np.zeros(8, np.uint8), 0)
    with pytest.raises(SizeMismatch):           # send 8 bytes vs recv 4 bytes
        ch.recv(4, 0)
    ch2 = Channel(FWD, 0, 2, 1024)
    ch2.send(np.zeros(8, np.uint8), 5)
    with pytest.raises(OrderError):
        ch2.recv(8, 4)
    ch3 = Channel(BWD, 1, 2, 64)
    ch3.send(np.ones(4, np.uint8), 0)
    ch3.send(np.ones(4, np.uint8), 1)
    with pytest.raises(WouldBlock):             # K = 2 slots both unconsumed
        ch3.send(np.ones(4, np.uint8), 2)
    ch3.recv(4, 0)
    ch3.send(np.ones(4, np.uint8), 2)
    with pytest.raises(WouldBlock):
        Channel(FWD, 0, 2, 64).recv(4, 0)       # nothing sent: rendezvous stays pending


def _masks(seed, n):
    cache = {}

    def mask(s, d, m):
        if (s, d, m) not in cache:
            cache[(s, d, m)] = P.proxy_mask(seed, 0, s, d, m, n)
        return cache[(s, d, m)]
    return mask


@pytest.mark.parametrize("S", [1, 2, 3, 5])
@pytest.mark.parametrize("M", [1, 3, 6])
@pytest.mark.parametrize("K", [1, 2, 3])
def test_xor_proxy_run_matches_closed_form(S, M, K):
    n = 1000 + 37 * S + M          # ragged size
    mask = _masks(42, n)
    src = lambda m: P.source_activation(42, 0, m, n)
    dsrc = lambda m: P.source_gradient(42, 0, m, n)
    Y, dX, chans, order = run_1f1b(S, M, K, xor_stage(mask, FWD), xor_stage(mask, BWD), src,
                                   dsrc, n, n, n)
    for m in range(M):
        y, g = xor_closed_form(S, m, src(m), dsrc(m), mask)
        assert np.array_equal(Y[m], y) and np.array_equal(dX[m], g)
    for (d, b), ch in chans.items():                # exactly once, in order
        assert [r[0] for r in ch.log] == list(range(1, M + 1))
        assert [r[1] for r in ch.log] == list(range(M))
        assert all(r[2] == n for r in ch.log)
    assert len(order) == 2 * S * M


def test_xor_proxy_detects_swaps():
    n = 256
    mask = _masks(42, n)
    x0, g0 = P.source_activation(42, 0, 0, n), P.source_gradient(42, 0, 0, n)
    y0, _ = xor_closed_form(3, 0, x0, g0, mask)
    y1, _ = xor_closed_form(3, 1, x0, g0, mask)
    assert not np.array_equal(y0, y1)     # mb 0's data with mb 1's masks is visible
    assert digest(y0) != digest(y1)
