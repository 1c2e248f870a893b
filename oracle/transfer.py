"""O3 — byte-level model of the stage-boundary ring transfer.  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2.2 P:L53 ("the source GPU first performs a device-to-device (D2D)
memory copy to move data from the user buffer into chunk buffer ... the receiver
performs a symmetric operation to copy the data into GPU memory") in the reading
DESIGN.md R7 fixes: the sender copies the user buffer straight into the receiver's
ring slot (one pass), the receiver copies the slot out into its user buffer.
Flow control and matching follow SPEC.md S:L395-397 (chunks in flight bounded by
slots; acknowledgement = receiver completion) and S:L355-361 (SizeMismatch).

Each receiving rank holds, per (boundary, direction), a ring of K slots, each a
64-byte header + payload.  Header (little-endian):
    u32 magic = 0x48435043 | u8 dir | u8 boundary | u16 0 |
    u64 bytes | u64 seq | i64 mb | u64 step | pad to 64 B
send(seq): needs credit >= seq - K, writes header + payload into slot seq % K.
recv(seq): checks magic, bytes (SIZE_MISMATCH), seq and mb (ORDER), copies the
payload out, sets credit = seq, appends (seq, mb, bytes, blake2b-128) to the log.

Pinned by tests/test_oracle_transfer.py: identity (delivered == sent, byte for
byte), exactly-once / in-order logs, the error cases, and the library special case
`bytes(payload)` copy; the GPU path is compared with this log and these bytes.
"""
from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import numpy as np

MAGIC = 0x48435043
HEADER_BYTES = 64
_HDR = struct.Struct("<IBBHQQqQ")   # 36 bytes, padded to 64
FWD, BWD = 0, 1


class TransferError(RuntimeError):
    code = "ERR"


class SizeMismatch(TransferError):
    code = "SIZE_MISMATCH"


class OrderError(TransferError):
    code = "ORDER"


class WouldBlock(TransferError):
    code = "WOULD_BLOCK"


def pack_header(direction: int, boundary: int, nbytes: int, seq: int, mb: int, step: int) -> bytes:
    raw = _HDR.pack(MAGIC, direction, boundary, 0, nbytes, seq, mb, step)
    return raw + bytes(HEADER_BYTES - len(raw))


def unpack_header(raw: bytes) -> dict:
    magic, d, bnd, _z, nb, seq, mb, step = _HDR.unpack(bytes(raw[:_HDR.size]))
    return dict(magic=magic, dir=d, boundary=bnd, bytes=nb, seq=seq, mb=mb, step=step)


def digest(payload: np.ndarray) -> str:
    return hashlib.blake2b(np.ascontiguousarray(payload).tobytes(), digest_size=16).hexdigest()


@dataclass
class Channel:
    """One (boundary, direction) connection: ring in receiver memory, credit in sender memory."""
    direction: int
    boundary: int
    K: int
    max_bytes: int
    headers: List[bytearray] = field(default_factory=list)
    slots: List[np.ndarray] = field(default_factory=list)
    send_seq: int = 0
    recv_seq: int = 0
    credit: int = 0                       # last consumed seq (lives on the sender)
    log: List[Tuple[int, int, int, str]] = field(default_factory=list)

    def __post_init__(self):
        self.headers = [bytearray(HEADER_BYTES) for _ in range(self.K)]
        self.slots = [np.zeros(self.max_bytes, np.uint8) for _ in range(self.K)]

    def send(self, payload: np.ndarray, mb: int, step: int = 0) -> int:
        payload = np.ascontiguousarray(payload, dtype=np.uint8).reshape(-1)
        n = payload.size
        if n > self.max_bytes:
            raise TransferError("TOO_LARGE")
        seq = self.send_seq + 1
        if self.credit < seq - self.K:
            raise WouldBlock(f"slot of seq {seq - self.K} not yet consumed")
        slot = seq % self.K
        self.headers[slot][:] = pack_header(self.direction, self.boundary, n, seq, mb, step)
        self.slots[slot][:n] = payload          # the one copy: user buffer -> peer slot
        self.send_seq = seq
        return seq

    def recv(self, nbytes: int, mb: int) -> np.ndarray:
        seq = self.recv_seq + 1
        if seq > self.send_seq:
            raise WouldBlock("nothing sent yet")
        slot = seq % self.K
        h = unpack_header(self.headers[slot])
        if h["magic"] != MAGIC:
            raise OrderError("bad magic")
        if h["bytes"] != nbytes:
            raise SizeMismatch(f"header bytes {h['bytes']} != recv bytes {nbytes}")
        if h["seq"] != seq or h["mb"] != mb:
            raise OrderError(f"header seq/mb {h['seq']}/{h['mb']} != expected {seq}/{mb}")
        out = self.slots[slot][:nbytes].copy()  # symmetric copy-out into the user buffer
        self.recv_seq = seq
        self.credit = seq
        self.log.append((seq, mb, nbytes, digest(out)))
        return out


def make_channels(S: int, K: int, max_bytes: int) -> Dict[Tuple[int, int], Channel]:
    """Channels of a pipeline of S stages: FWD on boundary b carries s=b -> b+1,
    BWD on boundary b carries b+1 -> b."""
    ch = {}
    for b in range(S - 1):
        ch[(FWD, b)] = Channel(FWD, b, K, max_bytes)
        ch[(BWD, b)] = Channel(BWD, b, K, max_bytes)
    return ch
