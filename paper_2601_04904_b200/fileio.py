"""BTA1 files to / from host and device (reference fileio.py:1-125).

Same format, reader semantics and error types as the reference:
``b"BTA1"``, little-endian u64 n, b, a, u8 dtype tag 0x10 (complex128), then
the raw blocks in the order diag, lower, upper, arrow_row, arrow_col, tip --
which is exactly this package's stacked storage order, so every kind is one
contiguous file region.

B200 additions: ``read_bta_device`` streams a file into a
``DeviceBta`` through two pinned staging buffers (the disk read of chunk k+1
overlaps the H2D copy of chunk k) and checks finiteness on the GPU;
``write_bta`` accepts a ``DeviceBta`` and streams it out the same way.  Host
reads go straight into the stacked arrays (``readinto``, optionally pinned).
"""

from __future__ import annotations

import os
import struct
import sys
from pathlib import Path

import numpy as np
import torch

from .errors import BadMagicError, ShapeInconsistencyError, TruncatedPayloadError
from .matrix import BtaMatrix

__all__ = ["read_bta", "write_bta", "read_bta_header", "read_bta_device", "payload_size", "MAGIC",
           "DTYPE_COMPLEX128"]

MAGIC = b"BTA1"
DTYPE_COMPLEX128 = 0x10
_HEADER = struct.Struct("<QQQB")
HEADER_SIZE = len(MAGIC) + _HEADER.size
KINDS = ("diag", "lower", "upper", "arrow_row", "arrow_col", "tip")
_STAGE_BYTES = 64 << 20


def _kind_shapes(n, b, a):
    return {"diag": (n, b, b), "lower": (n - 1, b, b), "upper": (n - 1, b, b), "arrow_row": (n, a, b),
            "arrow_col": (n, b, a), "tip": (a, a)}


def payload_size(n: int, b: int, a: int) -> int:
    """Payload size in bytes for the given shape (fileio.py:56-59)."""
    return 16 * (n * b * b + 2 * (n - 1) * b * b + 2 * n * a * b + a * a)


def _parse_header(head: bytes) -> tuple[int, int, int]:
    """fileio.py:78-90: magic, then truncation, dtype tag, shape checks."""
    if len(head) < len(MAGIC) or head[: len(MAGIC)] != MAGIC:
        raise BadMagicError(f"bad magic: expected {MAGIC!r}, got {head[:4]!r}")
    if len(head) < HEADER_SIZE:
        raise TruncatedPayloadError("file ends inside the header")
    n, b, a, tag = _HEADER.unpack(head[len(MAGIC):HEADER_SIZE])
    if tag != DTYPE_COMPLEX128:
        raise ShapeInconsistencyError(f"unknown dtype tag 0x{tag:02x}")
    if n < 1 or b < 1:
        raise ShapeInconsistencyError(f"invalid shape in header (n={n}, b={b}, a={a})")
    return n, b, a


def read_bta_header(path) -> tuple[int, int, int]:
    """Read and validate only the header; returns ``(n, b, a)``."""
    with open(path, "rb") as fh:
        return _parse_header(fh.read(HEADER_SIZE))


def _open_checked(path):
    """Open, parse the header and check the payload size (fileio.py:93-118)."""
    fh = open(path, "rb")
    try:
        n, b, a = _parse_header(fh.read(HEADER_SIZE))
        expected = payload_size(n, b, a)
        have = os.fstat(fh.fileno()).st_size - HEADER_SIZE
        if have < expected:
            raise TruncatedPayloadError(f"payload has {have} bytes, header requires {expected}")
        if have > expected:
            raise ShapeInconsistencyError(f"payload has {have} bytes, header requires exactly {expected}")
    except BaseException:
        fh.close()
        raise
    return fh, n, b, a


def read_bta(path, *, pinned: bool = False) -> BtaMatrix:
    """Read a BTA1 file into a host BtaMatrix (``pinned``: page-locked).

    Raises BadMagicError, TruncatedPayloadError, ShapeInconsistencyError for
    a wrong magic, a short payload, and an invalid header / oversized or
    non-finite payload, as the reference does."""
    fh, n, b, a = _open_checked(path)
    with fh:
        m = BtaMatrix.zeros(n, b, a, pinned=pinned, zero=False)
        for k, arr in m.stacked().items():
            if arr.size:
                view = memoryview(arr.reshape(-1).view(np.uint8))
                got = fh.readinto(view)
                if got != arr.nbytes:  # file shrank underneath us
                    raise TruncatedPayloadError(f"payload ended inside {k}")
    if sys.byteorder == "big":  # the payload is little-endian
        for arr in m.stacked().values():
            arr.byteswap(inplace=True)
    if any(not np.isfinite(arr).all() for arr in m.stacked().values()):
        raise ShapeInconsistencyError("payload contains non-finite entries")
    return m


def write_bta(m, path) -> None:
    """Write a host BtaMatrix or a DeviceBta losslessly (fileio.py:62-69);
    ``read_bta`` restores it bit for bit."""
    from .device import DeviceBta

    path = Path(path)
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(_HEADER.pack(m.n, m.b, m.a, DTYPE_COMPLEX128))
        if isinstance(m, DeviceBta):
            _write_device(m, fh)
            return
        for k in KINDS:
            arr = m.stacked()[k]
            if arr.size:
                fh.write(np.ascontiguousarray(arr, dtype="<c16").tobytes())


def _stages(nbytes):
    size = max(16, min(_STAGE_BYTES, nbytes))
    return [torch.empty(size, dtype=torch.uint8, pin_memory=True) for _ in range(2)]


def _regions(m):
    """(kind, flat uint8 device view) in file order."""
    out = []
    for k in KINDS:
        t = getattr(m, k)
        if t.numel():
            out.append((k, t.reshape(-1).view(torch.uint8)))
    return out


def read_bta_device(path, device=None):
    """Stream a BTA1 file into a DeviceBta: the file is read into two pinned
    staging buffers in turn while the other one's H2D copy runs; finiteness
    is checked on the device.  Same errors as ``read_bta``."""
    from .device import DeviceBta

    fh, n, b, a = _open_checked(path)
    with fh:
        X = DeviceBta.empty(n, b, a, device, zero=False)
        regions = _regions(X)
        stages = _stages(payload_size(n, b, a))
        copy = torch.cuda.Stream(X.device)
        done = [None, None]
        i = 0
        for k, dst in regions:
            off, total = 0, dst.numel()
            while off < total:
                buf = stages[i]
                if done[i] is not None:
                    done[i].synchronize()  # the staging buffer's previous copy finished
                step = min(buf.numel(), total - off)
                got = fh.readinto(memoryview(buf.numpy())[:step])
                if got != step:
                    raise TruncatedPayloadError(f"payload ended inside {k}")
                with torch.cuda.stream(copy):
                    dst[off:off + step].copy_(buf[:step], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(copy)
                done[i] = ev
                off += step
                i ^= 1
        torch.cuda.current_stream(X.device).wait_stream(copy)
    finite = torch.stack([torch.isfinite(getattr(X, k)).all() for k in KINDS if getattr(X, k).numel()]).all()
    if not bool(finite):
        raise ShapeInconsistencyError("payload contains non-finite entries")
    return X


def _write_device(m, fh):
    """D2H through two pinned staging buffers; the file write of chunk k
    overlaps the copy of chunk k+1."""
    nbytes = sum(getattr(m, k).numel() * 16 for k in KINDS)
    stages = _stages(nbytes)
    copy = torch.cuda.Stream(m.device)
    copy.wait_stream(torch.cuda.current_stream(m.device))
    pending = []  # (event, buf, step)
    i = 0

    def drain(keep):
        while len(pending) > keep:
            ev, buf, step = pending.pop(0)
            ev.synchronize()
            fh.write(memoryview(buf.numpy())[:step])

    for _, src in _regions(m):
        off, total = 0, src.numel()
        while off < total:
            buf = stages[i]
            drain(1)  # the buffer we are about to refill has been written
            step = min(buf.numel(), total - off)
            with torch.cuda.stream(copy):
                buf[:step].copy_(src[off:off + step], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            pending.append((ev, buf, step))
            off += step
            i ^= 1
    drain(0)
