"""Block kernels of the drop-in boundary (mirrors btasel/kernels.py).

``block_multiply_acc`` / ``mm`` and ``block_inverse`` run on the B200
through the C ABI (grouped complex128 DMMA GEMM and the blocked
Gauss-Jordan inverse).  ``OpCounter`` is the reference's shape-class tally;
the sweeps fill it with the reference's *logical* per-step inventory
(``record_sweep``) since the device executes fused multi-term products.
"""

from __future__ import annotations

import ctypes
from collections import Counter
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .errors import ShapeMismatchError

COMPLEX = np.complex128

__all__ = ["OpCounter", "block_multiply_acc", "mm", "block_inverse", "record_sweep"]


@dataclass
class OpCounter:
    """Tally of block operations keyed by operand shape class (kernels.py:37-96)."""

    b: int
    a: int = 0
    gemm_by_shape: Counter = field(default_factory=Counter)
    lu_count: int = 0
    trsm_count: int = 0
    inv_count: int = 0

    def _classify(self, d: int) -> str:
        if d == self.b:
            return "b"
        if d == self.a:
            return "a"
        return "?"

    def record_gemm(self, m: int, k: int, n: int) -> None:
        if m == 0 or k == 0 or n == 0:
            return
        self.gemm_by_shape[self._classify(m) + self._classify(k) + self._classify(n)] += 1

    def total_gemms(self) -> int:
        return sum(self.gemm_by_shape.values())

    def copy(self) -> "OpCounter":
        return OpCounter(self.b, self.a, Counter(self.gemm_by_shape), self.lu_count, self.trsm_count,
                         self.inv_count)

    def merge(self, other: "OpCounter") -> None:
        self.gemm_by_shape.update(other.gemm_by_shape)
        self.lu_count += other.lu_count
        self.trsm_count += other.trsm_count
        self.inv_count += other.inv_count

    def as_dict(self) -> dict:
        d = {f"gemm_{k}": v for k, v in sorted(self.gemm_by_shape.items())}
        d.update(lu=self.lu_count, trsm=self.trsm_count, inv=self.inv_count)
        return d


# Logical product inventory of the reference sweeps, as (count at n=1,
# increment per extra diagonal block) with symbolic classes over {b, a}.
# Derived from rgf.py:104-123, 237-318, 164-197, 440-487 (and checked
# against the reference's OpCounter by tests/test_host_logic.py).
_SWEEP_TABLE = {
    ("si", False, "forward"): ({}, {"bbb": 2}),
    ("si", False, "backward"): ({}, {"bbb": 5}),
    ("siq", False, "forward"): ({}, {"bbb": 8}),
    ("siq", False, "backward"): ({"bbb": 2}, {"bbb": 18}),
    ("si", True, "forward"): ({"aba": 1, "bba": 1}, {"aba": 1, "abb": 1, "bba": 2, "bbb": 2}),
    ("si", True, "backward"): ({"aab": 1, "abb": 1, "baa": 1, "bab": 1, "bba": 1, "bbb": 1},
                               {"aab": 1, "abb": 2, "baa": 1, "bab": 3, "bba": 2, "bbb": 6}),
    ("siq", True, "forward"): ({"aba": 4, "abb": 2}, {"aba": 4, "abb": 5, "bba": 5, "bbb": 8}),
    ("siq", True, "backward"): ({"aaa": 2, "aab": 4, "abb": 4, "baa": 3, "bab": 4, "bba": 4, "bbb": 9},
                                {"aab": 4, "abb": 8, "baa": 3, "bab": 11, "bba": 7, "bbb": 26}),
}


def _classify_label(label: str, b: int, a: int, counter: OpCounter) -> str:
    dims = {"b": b, "a": a}
    return "".join(counter._classify(dims[ch]) for ch in label)


def record_sweep(counter: OpCounter | None, n: int, b: int, a: int, mode: str, phase: str) -> None:
    """Add the reference's logical counts of one forward/backward sweep."""
    if counter is None:
        return
    base, step = _SWEEP_TABLE[(mode, a > 0, phase)]
    for label in set(base) | set(step):
        cnt = base.get(label, 0) + (n - 1) * step.get(label, 0)
        if cnt and not ("a" in label and a == 0):
            counter.gemm_by_shape[_classify_label(label, b, a, counter)] += cnt
    if phase == "forward":
        inv = n + (1 if a > 0 else 0)
        counter.lu_count += inv
        counter.inv_count += inv
        counter.trsm_count += 2 * inv


# ---------------------------------------------------------------------------
# GPU-backed kernels
# ---------------------------------------------------------------------------


def _as_block(x):
    if isinstance(x, torch.Tensor):
        if x.ndim != 2:
            raise ShapeMismatchError(f"expected a 2-d block, got ndim={x.ndim}")
        return x
    x = np.asarray(x, dtype=COMPLEX)
    if x.ndim != 2:
        raise ShapeMismatchError(f"expected a 2-d block, got ndim={x.ndim}")
    return x


def _dev(x, device):
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.complex128).contiguous()
    return torch.from_numpy(np.ascontiguousarray(x)).to(device)


def block_multiply_acc(c, a, b, *, alpha=1.0, beta=0.0, trans_a=False, trans_b=False, counter=None):
    """Return ``beta*c + alpha*op(a) @ op(b)`` computed on the GPU
    (kernels.py:106-154).  numpy in -> numpy out; CUDA tensors in -> CUDA
    tensor out."""
    a, b = _as_block(a), _as_block(b)
    m, k = (a.shape[1], a.shape[0]) if trans_a else (a.shape[0], a.shape[1])
    kb, n = (b.shape[1], b.shape[0]) if trans_b else (b.shape[0], b.shape[1])
    if k != kb:
        raise ShapeMismatchError(
            f"inner dimensions disagree: op(a) is {(m, k)}, op(b) is {(kb, n)}")
    if c is not None:
        c = _as_block(c)
        if tuple(c.shape) != (m, n):
            raise ShapeMismatchError(f"accumulator shape {tuple(c.shape)} does not match product shape {(m, n)}")
    if counter is not None:
        counter.record_gemm(m, k, n)
    on_device = isinstance(a, torch.Tensor) and a.is_cuda
    ctx = _native.Context.get(a.device.index if on_device else None)
    device = torch.device("cuda", ctx.device)
    da, db = _dev(a, device), _dev(b, device)
    dc = _dev(c, device) if (c is not None and beta != 0.0) else None
    out = torch.empty((m, n), dtype=torch.complex128, device=device)
    al, be = complex(alpha), complex(beta)
    ctx.bind_stream()
    ctx.call("bsel_block_multiply_acc", ctypes.c_void_p(out.data_ptr() if out.numel() else None), n,
             ctypes.c_void_p(dc.data_ptr() if dc is not None and dc.numel() else None), n,
             ctypes.c_void_p(da.data_ptr() if da.numel() else None), int(da.shape[1]), int(trans_a),
             ctypes.c_void_p(db.data_ptr() if db.numel() else None), int(db.shape[1]), int(trans_b),
             m, n, k, al.real, al.imag, be.real, be.imag)
    if on_device:
        return out
    return out.cpu().numpy()


def mm(a, b, counter=None, *, ta=False, tb=False):
    """``op(a) @ op(b)`` with counting; op = conjugate transpose (kernels.py:157-166)."""
    return block_multiply_acc(None, a, b, trans_a=ta, trans_b=tb, counter=counter)


def block_inverse(a, counter=None):
    """Explicit inverse on the GPU (kernels.py:220-236): blocked Gauss-Jordan
    with pivoted leaves and an exact partial-pivoting fallback.

    Raises SingularBlockError(index = pivot row) iff partial pivoting meets
    an exactly zero pivot.
    """
    a = _as_block(a)
    if a.shape[0] != a.shape[1]:
        raise ShapeMismatchError(f"LU requires a square block, got {tuple(a.shape)}")
    if counter is not None:
        counter.lu_count += 1
    n = a.shape[0]
    on_device = isinstance(a, torch.Tensor) and a.is_cuda
    if n == 0:
        if counter is not None:
            counter.inv_count += 1
            counter.trsm_count += 2
        return torch.empty((0, 0), dtype=torch.complex128, device=a.device) if on_device else \
            np.empty((0, 0), dtype=COMPLEX)
    ctx = _native.Context.get(a.device.index if on_device else None)
    device = torch.device("cuda", ctx.device)
    da = _dev(a, device)
    out = torch.empty((n, n), dtype=torch.complex128, device=device)
    ctx.bind_stream()
    ctx.call("bsel_block_inverse", ctypes.c_void_p(da.data_ptr()), n, ctypes.c_void_p(out.data_ptr()), n, n)
    if counter is not None:
        counter.inv_count += 1
        counter.trsm_count += 2
    return out if on_device else out.cpu().numpy()
