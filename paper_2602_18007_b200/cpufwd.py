"""ctypes binding of libppcb.so (include/ppcb.h): the CPU-Forwarding baseline B1 (pinned
/dev/shm ring, chunked D2H -> host flags -> H2D, `channels` host threads).  Baseline only —
the product path (libppc) never calls it."""
from __future__ import annotations

import ctypes as C
import os

from . import HERE, _check, _ptr, _stream

_PATH = os.path.join(HERE, "libppcb.so")
if not os.path.exists(_PATH):
    raise ImportError(f"{_PATH} is missing: build it with `python paper_2602_18007_b200/build.py`")
_lib = C.CDLL(_PATH)
_vp = C.c_void_p
_lib.ppcb_create.restype = C.c_int
_lib.ppcb_create.argtypes = [C.c_char_p, C.c_int, C.c_size_t, C.c_size_t, C.c_int, C.c_int, C.c_int,
                             C.c_uint, C.POINTER(_vp)]
for n, a in [("ppcb_connect", [_vp]), ("ppcb_destroy", [_vp]),
             ("ppcb_send", [_vp, _vp, C.c_size_t, C.c_longlong, _vp]),
             ("ppcb_recv", [_vp, _vp, C.c_size_t, C.c_longlong, _vp])]:
    getattr(_lib, n).restype = C.c_int
    getattr(_lib, n).argtypes = a


class CpuFwdLink:
    """One directed link of a pair: the sender side creates the shared ring."""

    def __init__(self, tag: str, is_sender: bool, max_msg: int, chunk: int = 4 << 20, K: int = 2,
                 channels: int = 4, device: int = 0, timeout_ms: int = 20000):
        h = C.c_void_p()
        _check(_lib.ppcb_create(tag.encode(), int(is_sender), max_msg, chunk, K, channels, device,
                                timeout_ms, C.byref(h)), "ppcb_create")
        self.h = h

    def connect(self):
        _check(_lib.ppcb_connect(self.h), "ppcb_connect")

    def send(self, buf, nbytes=None, mb=0, stream=None):
        p, n = _ptr(buf)
        _check(_lib.ppcb_send(self.h, p, n if nbytes is None else nbytes, mb, _stream(stream)),
               "ppcb_send")

    def recv(self, buf, nbytes=None, mb=0, stream=None):
        p, n = _ptr(buf)
        _check(_lib.ppcb_recv(self.h, p, n if nbytes is None else nbytes, mb, _stream(stream)),
               "ppcb_recv")

    def destroy(self):
        if self.h:
            _lib.ppcb_destroy(self.h)
            self.h = None
