"""C-ABI library checks that need no GPU: libppc.so loads, exports every symbol
include/ppc.h declares, the pure schedule generator equals the oracle, and the host
control plane (grid validation, DCBS groups, blob exchange, error codes) behaves.
Host-only comms (cuda_device = -1) touch no device memory."""
import ctypes
import os
import re

import pytest

import paper_2602_18007_b200 as ppc
from oracle.groups import build_groups
from oracle.schedule import schedule_1f1b

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ppc[b]?_[a-z0-9_]+)\s*\(", src)) - {"ppc_stage_fn"})


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(ppc.lib_path())
    names = _declared("ppc.h")
    assert "ppc_pp_send" in names and "ppc_step_1f1b" in names and len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n


def test_struct_layouts_match_the_binding():
    lib = ctypes.CDLL(ppc.lib_path())
    lib.ppc_struct_size.restype = ctypes.c_size_t
    lib.ppc_struct_size.argtypes = [ctypes.c_int]
    for which, cls in enumerate([ppc.Config, ppc.Step, ppc.Record, ppc.Op, ppc.Slot]):
        assert lib.ppc_struct_size(which) == ctypes.sizeof(cls), cls.__name__
    assert lib.ppc_struct_size(7) == 0


def test_schedule_matches_oracle():
    for S in range(1, 9):
        for s in range(S):
            for M in range(1, 33):
                assert ppc.schedule_1f1b(S, s, M) == schedule_1f1b(S, s, M)
    with pytest.raises(ppc.PpcError) as e:
        ppc.schedule_1f1b(2, 2, 4)
    assert e.value.name == "INVALID_ARG"


def test_status_strings():
    for i, name in enumerate(ppc.STATUS):
        assert ppc.status_str(i) == ("PPC_OK" if i == 0 else "PPC_ERR_" + name)


def test_create_errors_host_only():
    cfg = ppc.make_config(tp=2, pp=2, dp=1)
    with pytest.raises(ppc.PpcError) as e:
        ppc.Comm(cfg, 8, 0, -1)
    assert e.value.name == "GRID_MISMATCH"
    with pytest.raises(ppc.PpcError) as e:
        ppc.Comm(cfg, 4, 4, -1)
    assert e.value.name == "RANK_OUT_OF_RANGE"
    bad = ppc.make_config(pp=2, chunk_bytes=1000)
    with pytest.raises(ppc.PpcError) as e:
        ppc.Comm(bad, 2, 0, -1)
    assert e.value.name == "INVALID_ARG"


@pytest.mark.parametrize("tp,pp,dp", [(1, 2, 1), (2, 4, 1), (2, 2, 2), (1, 8, 1)])
def test_groups_match_oracle(tp, pp, dp):
    world = tp * pp * dp
    cfg = ppc.make_config(tp=tp, pp=pp, dp=dp)
    ref = build_groups(world, tp, pp, dp)
    comms = [ppc.Comm(cfg, world, r, -1) for r in range(world)]
    blobs = [c.export() for c in comms]
    for r, c in enumerate(comms):
        c.connect(blobs)
        for g, kind in ((ppc.GROUP_TP, "tp"), (ppc.GROUP_DP, "dp"), (ppc.GROUP_PP, "pp")):
            mem, be = c.group(g)
            assert mem in ref[kind] and r in mem
            assert be == (ppc.BACKEND_PEER if kind == "pp" else ppc.BACKEND_NCCL)
    for c in comms:
        c.destroy()


def test_host_only_data_path_is_state_error():
    cfg = ppc.make_config(pp=2)
    comms = [ppc.Comm(cfg, 2, r, -1) for r in range(2)]
    blobs = [c.export() for c in comms]
    for c in comms:
        c.connect(blobs)
    assert comms[0].pp_send(ppc.BWD, 0, 0, 0) == ppc.STATUS.index("NO_NEIGHBOR")
    assert comms[1].pp_send(ppc.FWD, 0, 0, 0) == ppc.STATUS.index("NO_NEIGHBOR")
    assert comms[0].pp_send(ppc.FWD, 0x1000, 64 << 20, 0) == ppc.STATUS.index("TOO_LARGE")
    assert comms[0].pp_send(ppc.FWD, 0, 16, 0) == ppc.STATUS.index("INVALID_ARG")  # null buf
    assert comms[0].pp_send(ppc.FWD, 0x1000, 16, -1) == ppc.STATUS.index("INVALID_ARG")
    assert comms[0].pp_send(ppc.FWD, 0x1000, 16, 0) == ppc.STATUS.index("STATE")  # no device
    # produce-in-place send: argument / state errors are synchronous and host-only
    sl = ctypes.byref(ppc.Slot())
    begin, end = ppc._send_begin, ppc._send_end
    assert begin(comms[0].h, ppc.BWD, 16, 0, None, sl) == ppc.STATUS.index("NO_NEIGHBOR")
    assert begin(comms[0].h, ppc.FWD, 0, 0, None, sl) == ppc.STATUS.index("INVALID_ARG")
    assert begin(comms[0].h, ppc.FWD, 16, -1, None, sl) == ppc.STATUS.index("INVALID_ARG")
    assert begin(comms[0].h, ppc.FWD, 16, 0, None, None) == ppc.STATUS.index("INVALID_ARG")
    assert begin(comms[0].h, ppc.FWD, 64 << 20, 0, None, sl) == ppc.STATUS.index("TOO_LARGE")
    assert begin(comms[0].h, ppc.FWD, 16, 0, None, sl) == ppc.STATUS.index("STATE")  # no device
    assert end(comms[0].h, ppc.FWD, 0, None) == ppc.STATUS.index("STATE")     # nothing open
    assert end(comms[0].h, 7, 0, None) == ppc.STATUS.index("INVALID_ARG")
    # batched receive: argument errors before anything is enqueued
    rb = ppc._recv_batch
    bufs = (ctypes.c_void_p * 17)(*([0x1000] * 17))
    sizes = (ctypes.c_size_t * 17)(*([16] * 17))
    big = (ctypes.c_size_t * 2)(16, 64 << 20)
    nul = (ctypes.c_void_p * 2)(0x1000, 0)
    assert rb(comms[1].h, ppc.FWD, bufs, sizes, 0, 0, None) == ppc.STATUS.index("INVALID_ARG")
    assert rb(comms[1].h, ppc.FWD, bufs, sizes, 17, 0, None) == ppc.STATUS.index("INVALID_ARG")
    assert rb(comms[1].h, ppc.FWD, bufs, sizes, 2, -1, None) == ppc.STATUS.index("INVALID_ARG")
    assert rb(comms[1].h, ppc.FWD, nul, sizes, 2, 0, None) == ppc.STATUS.index("INVALID_ARG")
    assert rb(comms[1].h, ppc.FWD, bufs, big, 2, 0, None) == ppc.STATUS.index("TOO_LARGE")
    assert rb(comms[0].h, ppc.FWD, bufs, sizes, 2, 0, None) == ppc.STATUS.index("NO_NEIGHBOR")
    assert rb(comms[1].h, ppc.FWD, bufs, sizes, 2, 0, None) == ppc.STATUS.index("STATE")
    for c in comms:
        c.destroy()


def test_connect_rejects_bad_blobs():
    cfg = ppc.make_config(pp=2)
    a, b = ppc.Comm(cfg, 2, 0, -1), ppc.Comm(cfg, 2, 1, -1)
    ba, bb = a.export(), b.export()
    with pytest.raises(ppc.PpcError) as e:        # blobs out of rank order
        a.connect([bb, ba])
    assert e.value.name == "RANK_OUT_OF_RANGE"
    with pytest.raises(ppc.PpcError) as e:        # neighbour slot holds our own blob
        fake = bytearray(ba)
        fake[8:12] = (1).to_bytes(4, "little")    # claims rank 1
        a.connect([ba, bytes(fake)])
    assert e.value.name == "SELF_SEND"
    other = ppc.Comm(ppc.make_config(pp=2, max_msg_bytes=1 << 20), 2, 1, -1)
    with pytest.raises(ppc.PpcError) as e:        # geometry differs
        a.connect([ba, other.export()])
    assert e.value.name == "INVALID_ARG"
    for c in (a, b, other):
        c.destroy()


def test_launch_counter_is_monotone():
    a = ppc.launch_count()
    assert a >= 0 and ppc.launch_count() >= a


def test_config_local_spin_field():
    cfg = ppc.make_config(pp=3, local_spin=1)
    assert cfg.local_spin == 1 and cfg.pp == 3
    comms = [ppc.Comm(cfg, 3, r, -1) for r in range(3)]     # host-only: accepted, no device
    for c in comms:
        c.destroy()
