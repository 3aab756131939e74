"""Device-resident BT(A) matrices: stacked torch complex128 tensors.

``DeviceBta`` is the zero-copy fast path of the boundary: its six tensors
are exactly the arrays of ``bsel_bta_t`` (include/btasel_b200.h).  Host
``BtaMatrix`` objects convert with one cudaMemcpy per block kind.
"""

from __future__ import annotations

import torch

from . import _native
from .errors import ShapeMismatchError
from .matrix import KINDS, BtaMatrix

__all__ = ["DeviceBta", "to_device", "to_host", "generate_dd_bta_device", "hermitianize_device", "kernel_launches"]


def _shapes(n, b, a):
    return {"diag": (n, b, b), "lower": (n - 1, b, b), "upper": (n - 1, b, b),
            "arrow_row": (n, a, b), "arrow_col": (n, b, a), "tip": (a, a)}


class DeviceBta:
    """Stacked device arrays of one BT(A) matrix (n, b, a)."""

    def __init__(self, n, b, a, tensors: dict):
        self.n, self.b, self.a = int(n), int(b), int(a)
        shapes = _shapes(self.n, self.b, self.a)
        for k, shp in shapes.items():
            t = tensors[k]
            if tuple(t.shape) != shp or t.dtype != torch.complex128 or not t.is_contiguous():
                raise ShapeMismatchError(f"{k}: expected contiguous complex128 {shp}, got {tuple(t.shape)}")
            setattr(self, k, t)

    @property
    def shape_params(self):
        return (self.n, self.b, self.a)

    @property
    def device(self):
        return self.diag.device

    def tensors(self) -> dict:
        return {k: getattr(self, k) for k in KINDS + ("tip",)}

    @classmethod
    def empty(cls, n, b, a, device=None, zero=True) -> "DeviceBta":
        dev = torch.device("cuda") if device is None else torch.device(device)
        mk = torch.zeros if zero else torch.empty
        return cls(n, b, a, {k: mk(s, dtype=torch.complex128, device=dev) for k, s in _shapes(n, b, a).items()})

    def clone(self) -> "DeviceBta":
        return DeviceBta(self.n, self.b, self.a, {k: t.clone() for k, t in self.tensors().items()})

    def desc(self) -> _native.Bta:
        d = _native.Bta()
        d.n, d.b, d.a = self.n, self.b, self.a
        for k, t in self.tensors().items():
            setattr(d, k, t.data_ptr() if t.numel() else None)
        return d

    def nbytes(self) -> int:
        return sum(t.numel() * 16 for t in self.tensors().values())

    def copy_from_host(self, m: BtaMatrix, non_blocking=True) -> "DeviceBta":
        if m.shape_params != self.shape_params:
            raise ShapeMismatchError("host/device shape mismatch")
        for k, arr in m.stacked().items():
            if arr.size:
                getattr(self, k).copy_(torch.from_numpy(arr), non_blocking=non_blocking)
        return self

    def copy_to_host(self, m: BtaMatrix, non_blocking=False) -> BtaMatrix:
        if m.shape_params != self.shape_params:
            raise ShapeMismatchError("host/device shape mismatch")
        for k, arr in m.stacked().items():
            if arr.size:
                torch.from_numpy(arr).copy_(getattr(self, k), non_blocking=non_blocking)
        return m

    def __repr__(self):
        return f"DeviceBta(n={self.n}, b={self.b}, a={self.a}, device={self.device})"


def to_device(m: BtaMatrix, device=None) -> DeviceBta:
    return DeviceBta.empty(m.n, m.b, m.a, device, zero=False).copy_from_host(m, non_blocking=False)


def to_host(d: DeviceBta, *, pinned=False) -> BtaMatrix:
    out = BtaMatrix.zeros(d.n, d.b, d.a, pinned=pinned)
    d.copy_to_host(out)
    return out


def generate_dd_bta_device(n, b, a, seed, dominance=1.5, device=None, *, out=None, _lane: int = 0) -> DeviceBta:
    """generate_dd_bta (matrix.py:224-284) computed on the GPU: the same
    splitmix64 stream bit for bit; the dominance shift's |row| sums are
    accumulated sequentially (host: numpy pairwise), so shifted diagonal
    entries may differ from the host generator in the last bit.  ``out``:
    an existing DeviceBta of the shape to overwrite (on the current stream).
    ``_lane`` (internal): native context lane -- callers generating from
    several host threads at once (EnergySweep pipes) need lanes of their own,
    because a context's stream binding is per context, not per thread."""
    import ctypes

    if n < 1 or b < 1 or a < 0:
        raise ValueError(f"invalid shape parameters (n={n}, b={b}, a={a})")
    if out is not None:
        if out.shape_params != (n, b, a):
            raise ShapeMismatchError("out has a different shape")
        device = out.device
    ctx = _native.Context.get(None if device is None else torch.device(device).index, lane=_lane)
    if out is None:
        out = DeviceBta.empty(n, b, a, torch.device("cuda", ctx.device), zero=False)
    d = out.desc()
    ctx.bind_stream()
    ctx.call("bsel_generate_dd_bta", ctypes.byref(d), int(seed) & 0xFFFFFFFFFFFFFFFF, float(dominance))
    return out


def hermitianize_device(m: DeviceBta, *, _lane: int = 0) -> DeviceBta:
    """In-place (m + m^H)/2 on the pattern (matrix.py:337-354); returns m.
    ``_lane``: see generate_dd_bta_device."""
    import ctypes

    ctx = _native.Context.get(m.device.index, lane=_lane)
    d = m.desc()
    ctx.bind_stream()
    ctx.call("bsel_hermitianize", ctypes.byref(d))
    return m


def kernel_launches() -> int:
    """Kernels launched by libbtasel_b200.so in this process."""
    return int(_native.load_library().bsel_kernel_launches())


def bind_host_to_device(index: int | None = None):
    """Bind the calling process to the CPUs local to CUDA device ``index``
    (NVML CPU affinity of the GPU's PCI address), so pinned host buffers
    allocated afterwards are first-touched on the GPU's NUMA node and the
    host<->device streams of concurrent GPUs do not cross the socket
    interconnect.  Returns the previous affinity set (pass it to
    os.sched_setaffinity to undo), or None when NVML is unavailable."""
    import os

    try:
        import pynvml
    except Exception:  # pragma: no cover - optional dependency
        return None
    if index is None:
        index = torch.cuda.current_device()
    try:
        prop = torch.cuda.get_device_properties(index)
        bus = f"{prop.pci_domain_id:08x}:{prop.pci_bus_id:02x}:{prop.pci_device_id:02x}.0"
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        ncpu = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {w * 64 + bit for w, m in enumerate(words) for bit in range(64) if (m >> bit) & 1}
        cpus &= set(range(ncpu))
        if not cpus:
            return None
        prev = os.sched_getaffinity(0)
        os.sched_setaffinity(0, cpus)
        return prev
    except Exception:  # NVML / affinity not permitted: leave the process as is
        return None
