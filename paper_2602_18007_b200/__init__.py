"""Thin ctypes binding of libppc (include/ppc.h): argument marshalling only.

Every step of the transfer path runs in libppc's sm_100a kernels; this module never
computes or copies data itself.  If libppc.so is missing this import fails loudly —
there is no CPU fallback (build with `python paper_2602_18007_b200/build.py` or
`__graft_entry__.build()`).

Names follow include/ppc.h (pp_send / pp_recv / schedule_1f1b / step_1f1b / DCBS
groups).  Pointers may be given as ints or as torch tensors (data_ptr / nbytes).
"""
from __future__ import annotations

import ctypes as C
import os

# More hardware queues than the default 8: each comm uses a compute stream plus two
# send streams (and CE channel streams); aliased queues only add false dependencies.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libppc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with "
                      "`python paper_2602_18007_b200/build.py` (no CPU fallback exists)")
_lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

# ---- status codes (ppc_status_t) -------------------------------------------------------
STATUS = ["OK", "INVALID_ARG", "GRID_MISMATCH", "RANK_OUT_OF_RANGE", "SELF_SEND", "NO_NEIGHBOR",
          "TOO_LARGE", "SIZE_MISMATCH", "ORDER", "TIMEOUT", "BACKEND", "CUDA", "NCCL", "STATE",
          "WOULD_BLOCK"]
OK, WOULD_BLOCK = 0, 14
FWD, BWD = 0, 1
ENGINE_SM, ENGINE_CE, ENGINE_PULL = 0, 1, 2
GROUP_TP, GROUP_DP, GROUP_PP = 0, 1, 2
BACKEND_NCCL, BACKEND_PEER, BACKEND_NONE = 0, 1, 2
BLOB_BYTES = 512


class PpcError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        self.name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{what}: PPC_ERR_{self.name}" if what else f"PPC_ERR_{self.name}")


class Config(C.Structure):
    _fields_ = [("tp", C.c_int), ("pp", C.c_int), ("dp", C.c_int),
                ("max_msg_bytes", C.c_size_t), ("ring_slots", C.c_int), ("channels", C.c_int),
                ("chunk_bytes", C.c_size_t), ("engine", C.c_int), ("cta_per_channel", C.c_int),
                ("timeout_ns", C.c_ulonglong), ("trace", C.c_int), ("zc_async", C.c_int),
                ("local_spin", C.c_int)]


class Op(C.Structure):
    _fields_ = [("kind", C.c_int), ("mb", C.c_int)]


class Record(C.Structure):
    _fields_ = [("t_start_ns", C.c_longlong), ("t_end_ns", C.c_longlong), ("src", C.c_int),
                ("dst", C.c_int), ("dir", C.c_int), ("kind", C.c_int), ("seq", C.c_longlong),
                ("mb", C.c_longlong), ("bytes", C.c_longlong)]


STAGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t,
                       C.c_size_t, C.c_void_p)


class Step(C.Structure):
    _fields_ = [("M", C.c_int), ("fwd_bytes", C.c_size_t), ("bwd_bytes", C.c_size_t),
                ("fwd", C.c_void_p), ("bwd", C.c_void_p), ("fwd_user", C.c_void_p),
                ("bwd_user", C.c_void_p), ("x", C.c_void_p), ("g", C.c_void_p),
                ("y", C.c_void_p), ("dx", C.c_void_p)]


class Slot(C.Structure):
    """ppc_slot_t: where a produce-in-place send writes (ppc_pp_send_begin)."""
    _fields_ = [("payload", C.c_void_p), ("flags", C.c_void_p), ("seq", C.c_ulonglong),
                ("bytes", C.c_size_t), ("chunk_bytes", C.c_size_t), ("n_chunks", C.c_uint)]


class XorCtx(C.Structure):
    _fields_ = [("seed", C.c_int), ("step", C.c_int), ("stage", C.c_int), ("dir", C.c_int)]


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_vp, _sz, _i, _ll = C.c_void_p, C.c_size_t, C.c_int, C.c_longlong
_create = _sig("ppc_create", _i, [C.POINTER(Config), _i, _i, _i, C.POINTER(_vp)])
_export = _sig("ppc_export", _i, [_vp, _vp, C.POINTER(_sz)])
_connect = _sig("ppc_connect", _i, [_vp, _vp, _sz, _vp, _i])
_nccl_id = _sig("ppc_nccl_unique_id", _i, [_vp])
_group = _sig("ppc_group", _i, [_vp, _i, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)])
_send = _sig("ppc_pp_send", _i, [_vp, _i, _vp, _sz, _ll, _vp])
_recv = _sig("ppc_pp_recv", _i, [_vp, _i, _vp, _sz, _ll, _vp])
_waitc = _sig("ppc_pp_wait_consumed", _i, [_vp, _i, _vp])
_send_begin = _sig("ppc_pp_send_begin", _i, [_vp, _i, _sz, _ll, _vp, C.POINTER(Slot)])
_send_end = _sig("ppc_pp_send_end", _i, [_vp, _i, _i, _vp])
_xor_send = _sig("ppc_stage_xor_send", _i, [C.POINTER(Slot), C.POINTER(XorCtx), _i, _vp, _sz,
                                             _vp])
_sched = _sig("ppc_schedule_1f1b", _i, [_i, _i, _i, C.POINTER(Op), C.POINTER(_i)])
_step = _sig("ppc_step_1f1b", _i, [_vp, C.POINTER(Step), _vp])
_step_local = _sig("ppc_step_1f1b_local", _i, [C.POINTER(_vp), _i, C.POINTER(Step), C.POINTER(_vp)])
_allreduce = _sig("ppc_allreduce", _i, [_vp, _i, _vp, _sz, _i, _vp])
_hx_allreduce = _sig("ppc_hetero_allreduce", _i, [_vp, _vp, _sz, _i, _vp])
_recv_batch = _sig("ppc_pp_recv_batch", _i, [_vp, _i, C.POINTER(_vp), C.POINTER(_sz), _i, _ll, _vp])
_recv_gather = _sig("ppc_pp_recv_gather", _i, [_vp, _i, _vp, _sz, _ll, _vp])
_graph_create = _sig("ppc_graph_create", _i, [C.POINTER(_vp), _i, C.POINTER(Step), C.POINTER(_vp),
                                              C.POINTER(_vp)])
_graph_launch = _sig("ppc_graph_launch", _i, [_vp])
_graph_destroy = _sig("ppc_graph_destroy", _i, [_vp])
_register = _sig("ppc_register", _i, [_vp, _vp, _sz, _vp, C.POINTER(_sz)])
_reg_import = _sig("ppc_register_import", _i, [_vp, _vp, _sz])
REG_BLOB_BYTES = 128
_poll = _sig("ppc_poll", _i, [_vp])
_err_info = _sig("ppc_error_info", _i, [_vp, C.POINTER(C.c_uint), C.POINTER(C.c_uint)])
_trace = _sig("ppc_trace", _i, [_vp, C.POINTER(Record), C.POINTER(_i)])
_ktimes = _sig("ppc_kernel_times", _i, [_vp, _i, C.POINTER(C.c_float), C.POINTER(_i)])
_set_trace = _sig("ppc_set_trace", _i, [_vp, _i])
_dbg_stamps = _sig("ppc_debug_stamps", _i, [_vp, C.POINTER(C.c_ulonglong), C.POINTER(_ll),
                                            C.POINTER(_i)])
_disconnect = _sig("ppc_disconnect", _i, [_vp])
_destroy = _sig("ppc_destroy", _i, [_vp])
_status_str = _sig("ppc_status_str", C.c_char_p, [_i])
_fill = _sig("ppc_fill_payload", _i, [_vp, _sz, _i, _i, _i, _i, _ll, _vp])
_launch_count = _sig("ppc_launch_count", C.c_ulonglong, [])
STAGE_XOR = C.cast(_lib.ppc_stage_xor, C.c_void_p).value   # ppc_stage_fn address


def launch_count() -> int:
    """Kernels libppc enqueued in this process so far (ppc_launch_count)."""
    return int(_launch_count())


def lib_path() -> str:
    return LIB_PATH


def status_str(st: int) -> str:
    return _status_str(st).decode()


def _check(st: int, what: str):
    if st != OK:
        raise PpcError(st, what)


def _ptr(x):
    """(address, nbytes or None) of an int / torch tensor / None."""
    if x is None:
        return 0, None
    if isinstance(x, int):
        return x, None
    if hasattr(x, "data_ptr"):
        return x.data_ptr(), x.numel() * x.element_size()
    raise TypeError(f"cannot take a device pointer of {type(x)}")


def _stream(s):
    if s is None:
        return 0
    if isinstance(s, int):
        return s
    return s.cuda_stream


def make_config(tp=1, pp=2, dp=1, max_msg_bytes=32 << 20, ring_slots=0, channels=1,
                chunk_bytes=1 << 20, engine=ENGINE_SM, cta_per_channel=0, timeout_ns=0,
                trace=0, zc_async=0, local_spin=0) -> Config:
    return Config(tp, pp, dp, max_msg_bytes, ring_slots, channels, chunk_bytes, engine,
                  cta_per_channel, timeout_ns, trace, zc_async, local_spin)


def schedule_1f1b(S: int, s: int, M: int):
    ops = (Op * (2 * M))()
    n = C.c_int(0)
    _check(_sched(S, s, M, ops, C.byref(n)), "ppc_schedule_1f1b")
    return [("F" if ops[i].kind == 0 else "B", ops[i].mb) for i in range(n.value)]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_nccl_id(buf), "ppc_nccl_unique_id")
    return buf.raw


class Comm:
    """One rank's ppc_comm_t."""

    def __init__(self, cfg: Config, world: int, rank: int, device: int):
        self.cfg, self.world, self.rank, self.device = cfg, world, rank, device
        h = C.c_void_p()
        _check(_create(C.byref(cfg), world, rank, device, C.byref(h)), "ppc_create")
        self.h = h

    # -- lifecycle
    def export(self) -> bytes:
        buf = C.create_string_buffer(BLOB_BYTES)
        n = C.c_size_t(BLOB_BYTES)
        _check(_export(self.h, buf, C.byref(n)), "ppc_export")
        return buf.raw[:n.value]

    def connect(self, blobs, nccl_ids=None):
        allb = b"".join(blobs)
        ids = b"".join(nccl_ids) if nccl_ids else b""
        _check(_connect(self.h, allb, BLOB_BYTES, ids if ids else None, len(nccl_ids or [])),
               "ppc_connect")

    def group(self, g: int):
        n = C.c_int(self.world)
        mem = (C.c_int * self.world)()
        be = C.c_int(0)
        _check(_group(self.h, g, mem, C.byref(n), C.byref(be)), "ppc_group")
        return list(mem[:n.value]), be.value

    def disconnect(self):
        if self.h:
            _check(_disconnect(self.h), "ppc_disconnect")

    def destroy(self):
        if self.h:
            _check(_destroy(self.h), "ppc_destroy")
            self.h = None

    # -- data path
    def pp_send(self, direction, buf, nbytes=None, mb=0, stream=None):
        p, n = _ptr(buf)
        nbytes = n if nbytes is None else nbytes
        return _send(self.h, direction, p, nbytes, mb, _stream(stream))

    def pp_recv(self, direction, buf, nbytes=None, mb=0, stream=None):
        p, n = _ptr(buf)
        nbytes = n if nbytes is None else nbytes
        return _recv(self.h, direction, p, nbytes, mb, _stream(stream))

    def send(self, *a, **k):
        _check(self.pp_send(*a, **k), "ppc_pp_send")

    def recv(self, *a, **k):
        _check(self.pp_recv(*a, **k), "ppc_pp_recv")

    def send_begin(self, direction, nbytes, mb=0, stream=None) -> Slot:
        """Produce-in-place send: returns the receiver's slot to write (ppc_pp_send_begin)."""
        sl = Slot()
        _check(_send_begin(self.h, direction, nbytes, mb, _stream(stream), C.byref(sl)),
               "ppc_pp_send_begin")
        return sl

    def send_end(self, direction, flags_released=False, stream=None):
        _check(_send_end(self.h, direction, int(bool(flags_released)), _stream(stream)),
               "ppc_pp_send_end")

    def xor_send(self, direction, ctx, mb, inp, nbytes, stream=None):
        """The XOR stage proxy fused with its send: begin, ppc_stage_xor_send, end."""
        sl = self.send_begin(direction, nbytes, mb, stream)
        p = _ptr(inp)[0] if inp is not None else None
        _check(_xor_send(C.byref(sl), C.byref(ctx), mb, p, nbytes, _stream(stream)),
               "ppc_stage_xor_send")
        self.send_end(direction, True, stream)

    def wait_consumed(self, direction, stream=None):
        _check(_waitc(self.h, direction, _stream(stream)), "ppc_pp_wait_consumed")

    def allreduce(self, g, tensor, nccl_dtype, stream=None):
        p, n = _ptr(tensor)
        _check(_allreduce(self.h, g, p, tensor.numel(), nccl_dtype, _stream(stream)),
               "ppc_allreduce")

    def recv_batch(self, direction, bufs, nbytes, mb0=0, stream=None):
        """The next len(bufs) messages of `direction` in one grid (ppc_pp_recv_batch);
        nbytes: one size for all, or a list."""
        n = len(bufs)
        sizes = list(nbytes) if isinstance(nbytes, (list, tuple)) else [nbytes] * n
        ps = (C.c_void_p * n)(*[_ptr(b)[0] for b in bufs])
        ss = (C.c_size_t * n)(*sizes)
        _check(_recv_batch(self.h, direction, ps, ss, n, mb0, _stream(stream)),
               "ppc_pp_recv_batch")

    def recv_gather(self, direction, buf, nbytes=None, mb=0, stream=None):
        """TP-sliced boundary: receive every TP sender's slice (pulled, fused all-gather)."""
        p, n = _ptr(buf)
        _check(_recv_gather(self.h, direction, p, n if nbytes is None else nbytes, mb,
                            _stream(stream)), "ppc_pp_recv_gather")

    def register(self, buf, nbytes=None) -> bytes:
        """Register a send buffer for zero-copy pulls; returns the blob for the neighbours."""
        p, n = _ptr(buf)
        out = C.create_string_buffer(REG_BLOB_BYTES)
        sz = C.c_size_t(REG_BLOB_BYTES)
        _check(_register(self.h, p, n if nbytes is None else nbytes, out, C.byref(sz)),
               "ppc_register")
        return out.raw

    def register_import(self, blob: bytes):
        _check(_reg_import(self.h, blob, len(blob)), "ppc_register_import")

    def hetero_allreduce(self, tensor, nccl_dtype, stream=None):
        """NCCL inside each stage's DP subgroup + leader exchange over the PP peer path."""
        p, _ = _ptr(tensor)
        _check(_hx_allreduce(self.h, p, tensor.numel(), nccl_dtype, _stream(stream)),
               "ppc_hetero_allreduce")

    def poll(self) -> int:
        return _poll(self.h)

    def error_info(self):
        """(status name, seq, info) of the latched device error, if any."""
        seq, info = C.c_uint(0), C.c_uint(0)
        st = _err_info(self.h, C.byref(seq), C.byref(info))
        return STATUS[st], seq.value, hex(info.value)

    def set_trace(self, trace: int):
        _check(_set_trace(self.h, trace), "ppc_set_trace")

    def kernel_times(self, kind: int, cap=4096):
        """Device ms of each send (0) / recv (1) launch since the last call (cfg.trace & 2)."""
        out = (C.c_float * cap)()
        n = C.c_int(cap)
        _check(_ktimes(self.h, kind, out, C.byref(n)), "ppc_kernel_times")
        return list(out[:n.value])

    def debug_stamps(self, cap=4096):
        """PPC_DBG_STAMPS receive-kernel stamps: list of (seq, dir, grid, [[4 stamps] per CTA])."""
        st = (C.c_ulonglong * (cap * 512))()
        meta = (C.c_longlong * (cap * 3))()
        n = C.c_int(cap)
        _check(_dbg_stamps(self.h, st, meta, C.byref(n)), "ppc_debug_stamps")
        out = []
        for i in range(n.value):
            g = meta[3 * i + 2]
            rows = [list(st[i * 512 + 4 * b: i * 512 + 4 * b + 4]) for b in range(g)]
            out.append((meta[3 * i], meta[3 * i + 1], g, rows))
        return out

    def trace(self, cap=8192):
        recs = (Record * cap)()
        n = C.c_int(cap)
        _check(_trace(self.h, recs, C.byref(n)), "ppc_trace")
        return [dict(t_start_ns=r.t_start_ns, t_end_ns=r.t_end_ns, src=r.src, dst=r.dst,
                     dir=r.dir, kind=r.kind, seq=r.seq, mb=r.mb, bytes=r.bytes)
                for r in recs[:n.value]]


class StepArgs:
    """Owns the ctypes arrays behind one ppc_step_t."""

    def __init__(self, M, fwd_bytes, bwd_bytes=None, fwd=None, bwd=None, fwd_user=None,
                 bwd_user=None, x=None, g=None, y=None, dx=None):
        self._keep = []
        self.st = Step()
        self.st.M = M
        self.st.fwd_bytes = fwd_bytes
        self.st.bwd_bytes = fwd_bytes if bwd_bytes is None else bwd_bytes
        self.st.fwd = self._fn(fwd)
        self.st.bwd = self._fn(bwd)
        self.st.fwd_user = self._user(fwd_user)
        self.st.bwd_user = self._user(bwd_user)
        self.st.x = self._arr(x)
        self.st.g = self._arr(g)
        self.st.y = self._arr(y)
        self.st.dx = self._arr(dx)

    def _fn(self, f):
        if f is None:
            return None
        if isinstance(f, int):
            return f
        cb = STAGE_FN(f)
        self._keep.append(cb)
        return C.cast(cb, C.c_void_p).value

    def _user(self, u):
        if u is None:
            return None
        if isinstance(u, int):
            return u
        self._keep.append(u)
        return C.addressof(u)

    def _arr(self, lst):
        if lst is None:
            return None
        a = (C.c_void_p * len(lst))(*[_ptr(t)[0] for t in lst])
        self._keep.append(a)
        return C.addressof(a)


def step_1f1b(comm: Comm, args: StepArgs, stream=None):
    _check(_step(comm.h, C.byref(args.st), _stream(stream)), "ppc_step_1f1b")


def step_1f1b_local(comms, args, streams):
    S = len(comms)
    hs = (C.c_void_p * S)(*[c.h.value for c in comms])
    steps = (Step * S)(*[a.st for a in args])
    ss = (C.c_void_p * S)(*[_stream(s) for s in streams])
    _check(_step_local(hs, S, steps, ss), "ppc_step_1f1b_local")


class StepGraph:
    """One 1F1B step captured into a CUDA graph (ppc_graph_create); launch() replays the next
    step.  comms/args/streams as for step_1f1b (one comm) or step_1f1b_local (S comms).
    Run one eager step before creating it (the step's buffers must exist)."""

    def __init__(self, comms, args, streams):
        comms, args, streams = list(comms), list(args), list(streams)
        self._keep = (comms, args)
        self._steps = (Step * len(args))(*[a.st for a in args])
        hs = (C.c_void_p * len(comms))(*[c.h.value for c in comms])
        ss = (C.c_void_p * len(streams))(*[_stream(s) for s in streams])
        h = C.c_void_p()
        _check(_graph_create(hs, len(comms), self._steps, ss, C.byref(h)), "ppc_graph_create")
        self.h = h

    def launch(self):
        _check(_graph_launch(self.h), "ppc_graph_launch")

    def destroy(self):
        if self.h:
            _check(_graph_destroy(self.h), "ppc_graph_destroy")
            self.h = None


def fill_payload(buf, nbytes=None, seed=42, step=0, boundary=0, direction=0, mb=0, stream=None):
    p, n = _ptr(buf)
    nbytes = n if nbytes is None else nbytes
    _check(_fill(p, nbytes, seed, step, boundary, direction, mb, _stream(stream)),
           "ppc_fill_payload")


# ---- process wiring (host control plane: bootstrap all-gather) ----------------------
def virtual_stages(cfg: Config, device=0):
    """S = cfg.pp virtual stages of one pipeline in this process (K11 path).  `device` is one
    device index for all stages, or a list with one device per stage (stages on different
    GPUs of one process: NVLink transfers ordered by events, used for profiling).  With
    cfg.local_spin the stages run the cross-process protocol instead (device spins; step
    each with step_1f1b)."""
    return local_comms(cfg, device)


def local_comms(cfg: Config, device=0):
    """Every rank of the cfg grid (tp * pp * dp comms, rank order) in this process, blobs
    exchanged in-process.  `device`: one index for all ranks or a list per rank."""
    world = cfg.tp * cfg.pp * cfg.dp
    devs = list(device) if isinstance(device, (list, tuple)) else [device] * world
    comms = [Comm(cfg, world, r, devs[r]) for r in range(world)]
    blobs = [c.export() for c in comms]
    for c in comms:
        c.connect(blobs)
    return comms


def register_local(comms, tensors_by_rank):
    """register_tensors for comms of one process: tensors_by_rank[r] are rank r's send
    buffers; every comm imports every registration (non-neighbours ignore them)."""
    blobs = [comms[r].register(t) for r in range(len(comms)) for t in (tensors_by_rank[r] or [])]
    for c in comms:
        for b in blobs:
            c.register_import(b)


def connect_distributed(cfg: Config, rank: int, world: int, device: int, pg=None,
                        with_nccl: bool = True) -> Comm:
    """One process per GPU: gloo all-gather of the blobs (Topology Awareness) and of
    NCCL ids for the TP/DP groups (DCBS)."""
    import torch.distributed as dist
    comm = Comm(cfg, world, rank, device)
    blobs = [None] * world
    dist.all_gather_object(blobs, comm.export(), group=pg)
    ids = None
    if with_nccl:
        mine = {}
        tp_m, _ = comm.group(GROUP_TP)
        dp_m, _ = comm.group(GROUP_DP)
        single = os.environ.get("PPC_NCCL_SINGLETON") == "1"   # tests: one-rank groups too
        if rank == min(tp_m) and (len(tp_m) > 1 or single):
            mine["tp"] = nccl_unique_id()
        if rank == min(dp_m) and (len(dp_m) > 1 or single):
            mine["dp"] = nccl_unique_id()
        allids = [None] * world
        dist.all_gather_object(allids, mine, group=pg)
        zero = bytes(128)
        ids = [allids[min(tp_m)].get("tp", zero), allids[min(dp_m)].get("dp", zero)]
    comm.connect(blobs, ids)
    return comm


def register_tensors(comm: Comm, tensors, pg=None):
    """Collective: register this rank's send buffers for zero-copy pulls and import every
    neighbour's registrations (gloo all-gather of the registration blobs)."""
    import torch.distributed as dist
    mine = [comm.register(t) for t in (tensors or [])]
    world = dist.get_world_size(pg)
    allb = [None] * world
    dist.all_gather_object(allb, mine, group=pg)
    for blobs in allb:
        for b in blobs:
            comm.register_import(b)
