"""Parity of EXACTLY what bench.py times (the timed configuration had no parity
test).  The tests build bench.py's own Pipeline (same comms, buffers, chunking, K, CUDA graph)
for the N = 1 headline — C2 [1,4096,4096] bf16, PP = 2, M = 8, identity stages, device X / G /
Y / DX, 128 KiB chunks, K = 3, the step replayed as a CUDA graph — in the direct single-copy
mode and on the intra-device ring, and compare ALL 8 Y and 8 DX byte for byte with the CPU
oracle's 1F1B byte simulation of the same step (oracle/proxy.run_1f1b on synth payloads)."""
import numpy as np
import pytest
import torch

import bench
from oracle.proxy import run_1f1b
from synth import payload as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def oracle_c2():
    wl = bench.resolve(bench.parse([]), 1)
    n, M = wl["msg_bytes"], wl["M"]
    ident = lambda s, m, x: x
    Y, DX, chans, _ = run_1f1b(2, M, wl["slots"], ident, ident,
                               lambda m: P.source_activation(42, 0, m, n),
                               lambda m: P.source_gradient(42, 0, m, n), n, n, n)
    return wl, Y, DX


@pytest.mark.parametrize("direct", [True, False])
def test_bench_n1_timed_step_matches_oracle(direct, oracle_c2):
    wl, Yo, DXo = oracle_c2
    assert (wl["pp"], wl["M"], wl["msg_bytes"], wl["chunk"], wl["slots"], wl["graph"]) == \
        (2, 8, 4096 * 4096 * 2, 128 << 10, 3, True)
    ctx = bench.Ctx()
    p = bench.Pipeline(ctx, wl, local_direct=direct)
    assert p.graph is not None
    for rep in range(3):                      # graph replays (warm-up + timed steps)
        for t in p.Y[1] + p.DX[0]:
            t.zero_()
        ms = p.timed(2)
        assert ms > 0
        assert p.outputs_ok()                 # bench.py's own device-side check agrees
        for m in range(wl["M"]):
            assert np.array_equal(p.Y[1][m].cpu().numpy(), Yo[m]), (rep, m)
            assert np.array_equal(p.DX[0][m].cpu().numpy(), DXo[m]), (rep, m)
    for c in p.comms:
        assert c.poll() == 0
    p.close()


def test_bench_outputs_check_detects_corruption(oracle_c2):
    """bench.py's outputs_checked must fail when a single byte of one output is wrong."""
    wl, _, _ = oracle_c2
    ctx = bench.Ctx()
    p = bench.Pipeline(ctx, {**wl, "graph": False})
    p.step()
    torch.cuda.synchronize()
    assert p.outputs_ok()
    p.DX[0][5][12345] ^= 1
    assert not p.outputs_ok()
    p.close()
