"""ctypes binding of libppctoy.so (include/ppc_toy.h): the C1 toy pipeline's stage compute
as ppc_stage_fn callbacks.  Marshalling only; fails loudly if the library is missing."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import HERE, PpcError, StepArgs, _check

_PATH = os.path.join(HERE, "libppctoy.so")
if not os.path.exists(_PATH):
    raise ImportError(f"{_PATH} is missing: build it with `python paper_2602_18007_b200/build.py`")
_lib = C.CDLL(_PATH)
_vp = C.c_void_p
_lib.ppc_toy_create.restype = C.c_int
_lib.ppc_toy_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_int, C.c_int,
                                C.POINTER(_vp)]
for name, args in [("ppc_toy_set_params", [_vp, _vp, _vp]), ("ppc_toy_get_params", [_vp, _vp, _vp]),
                   ("ppc_toy_set_data", [_vp, _vp]), ("ppc_toy_step_end", [_vp, _vp]),
                   ("ppc_toy_loss", [_vp, _vp, C.POINTER(C.c_double)]),
                   ("ppc_toy_destroy", [_vp])]:
    f = getattr(_lib, name)
    f.restype = C.c_int
    f.argtypes = args
_lib.ppc_toy_boundary_bytes.restype = C.c_size_t
_lib.ppc_toy_boundary_bytes.argtypes = [_vp]
TOY_FWD = C.cast(_lib.ppc_toy_fwd, C.c_void_p).value
TOY_BWD = C.cast(_lib.ppc_toy_bwd, C.c_void_p).value
_fwd = _lib.ppc_toy_fwd
_fwd.restype = C.c_int
_fwd.argtypes = [_vp, C.c_int, _vp, _vp, C.c_size_t, C.c_size_t, _vp]
_bwd = _lib.ppc_toy_bwd
_bwd.restype = C.c_int
_bwd.argtypes = [_vp, C.c_int, _vp, _vp, C.c_size_t, C.c_size_t, _vp]


def _s(stream):
    return 0 if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)


class ToyStage:
    """One stage (0 or 1) of the C1 toy model on `device`."""

    def __init__(self, stage, rows, width, M, lr, bf16, device, W2, b2, data):
        h = C.c_void_p()
        _check(_lib.ppc_toy_create(stage, rows, width, M, lr, int(bf16), device, C.byref(h)),
               "ppc_toy_create")
        self.h, self.stage, self.M = h, stage, M
        self.rows, self.width = rows, width
        W = np.ascontiguousarray(np.stack(W2), dtype=np.float32)
        b = np.ascontiguousarray(np.stack(b2), dtype=np.float32)
        _check(_lib.ppc_toy_set_params(h, W.ctypes.data, b.ctypes.data), "ppc_toy_set_params")
        d = np.ascontiguousarray(np.stack(data), dtype=np.float32)
        _check(_lib.ppc_toy_set_data(h, d.ctypes.data), "ppc_toy_set_data")

    @property
    def boundary_bytes(self):
        return _lib.ppc_toy_boundary_bytes(self.h)

    def step_args(self):
        return StepArgs(self.M, self.boundary_bytes, self.boundary_bytes, fwd=TOY_FWD,
                        bwd=TOY_BWD, fwd_user=self.h.value, bwd_user=self.h.value)

    def fwd(self, mb, inp, out, stream=None):
        st = _fwd(self.h, mb, inp or 0, out or 0, self.boundary_bytes, self.boundary_bytes, _s(stream))
        if st:
            raise PpcError(st, "ppc_toy_fwd")

    def bwd(self, mb, inp, out, stream=None):
        st = _bwd(self.h, mb, inp or 0, out or 0, self.boundary_bytes, self.boundary_bytes, _s(stream))
        if st:
            raise PpcError(st, "ppc_toy_bwd")

    def step_end(self, stream=None):
        _check(_lib.ppc_toy_step_end(self.h, _s(stream)), "ppc_toy_step_end")

    def loss(self, stream=None) -> float:
        v = C.c_double()
        _check(_lib.ppc_toy_loss(self.h, _s(stream), C.byref(v)), "ppc_toy_loss")
        return v.value

    def params(self):
        W = np.empty((2, self.width, self.width), np.float32)
        b = np.empty((2, self.width), np.float32)
        _check(_lib.ppc_toy_get_params(self.h, W.ctypes.data, b.ctypes.data), "ppc_toy_get_params")
        return W, b

    def destroy(self):
        if self.h:
            _lib.ppc_toy_destroy(self.h)
            self.h = None
