"""Dense oracle on the GPU (reference baselines.py:35-81).

``dense_solve`` expands the system to an N x N dense matrix on the device
(N = n*b + a <= guard, default 4096 as in the reference), inverts it with
the library's blocked Gauss-Jordan kernel, forms A^-1 B A^-H with the
grouped DMMA GEMM, and masks both to the pattern.  It is the independent
GPU cross-check of the RGF sweeps at sizes the CPU oracle is slow for; it
shares no code path with the sweeps except the two kernels.
"""

from __future__ import annotations

import ctypes
from time import perf_counter

import torch

from . import _native
from .device import DeviceBta, to_device, to_host
from .errors import DenseGuardError, ShapeMismatchError
from .kernels import OpCounter
from .matrix import SelectedSolution

__all__ = ["dense_solve", "dense_device", "mask_device", "DEFAULT_DENSE_GUARD"]

DEFAULT_DENSE_GUARD = 4096


def dense_device(m: DeviceBta) -> torch.Tensor:
    """N x N dense expansion on the device, zeros off the pattern
    (matrix.py:292-306)."""
    n, b, a = m.shape_params
    nb = n * b
    big = torch.zeros((nb + a, nb + a), dtype=torch.complex128, device=m.device)
    blocks = big[:nb, :nb].view(n, b, n, b)
    idx = torch.arange(n, device=m.device)
    blocks[idx, :, idx, :] = m.diag
    if n > 1:
        blocks[idx[1:], :, idx[:-1], :] = m.lower
        blocks[idx[:-1], :, idx[1:], :] = m.upper
    if a:
        big[nb:, :nb] = m.arrow_row.permute(1, 0, 2).reshape(a, nb)
        big[:nb, nb:] = m.arrow_col.reshape(nb, a)
        big[nb:, nb:] = m.tip
    return big


def mask_device(dense: torch.Tensor, shape) -> DeviceBta:
    """The in-pattern blocks of a dense device array (matrix.py:309-334)."""
    n, b, a = shape
    nb = n * b
    if tuple(dense.shape) != (nb + a, nb + a):
        raise ShapeMismatchError(f"dense array has shape {tuple(dense.shape)}, expected {(nb + a,) * 2}")
    out = DeviceBta.empty(n, b, a, dense.device, zero=False)
    blocks = dense[:nb, :nb].reshape(n, b, n, b)
    idx = torch.arange(n, device=dense.device)
    out.diag.copy_(blocks[idx, :, idx, :])
    if n > 1:
        out.lower.copy_(blocks[idx[1:], :, idx[:-1], :])
        out.upper.copy_(blocks[idx[:-1], :, idx[1:], :])
    if a:
        out.arrow_row.copy_(dense[nb:, :nb].reshape(a, n, b).permute(1, 0, 2))
        out.arrow_col.copy_(dense[:nb, nb:].reshape(n, b, a))
        out.tip.copy_(dense[nb:, nb:])
    return out


def _gemm(ctx, out, x, y, trans_y=False):
    N = out.shape[0]
    ctx.call("bsel_block_multiply_acc", ctypes.c_void_p(out.data_ptr()), N, None, N,
             ctypes.c_void_p(x.data_ptr()), N, 0, ctypes.c_void_p(y.data_ptr()), N, int(trans_y),
             N, N, N, 1.0, 0.0, 0.0, 0.0)


def dense_solve(a, b=None, mode=None, *, guard: int | None = None, counter: OpCounter | None = None,
                timings: dict | None = None) -> SelectedSolution:
    """Dense reference solve masked to the pattern, on the GPU
    (baselines.py:35-81).  Host BtaMatrix in -> host out; DeviceBta in ->
    DeviceBta out.  Refuses N > guard (DenseGuardError)."""
    if mode is None:
        mode = "si" if b is None else "siq"
    if mode == "siq" and b is None:
        raise ValueError("mode 'siq' requires a right-hand side")
    if b is not None and b.shape_params != a.shape_params:
        raise ShapeMismatchError("right-hand side shape differs from system shape")
    n, bs, asz = a.shape_params
    total = n * bs + asz
    if total > (DEFAULT_DENSE_GUARD if guard is None else guard):
        raise DenseGuardError(f"dense path refused: total size {total} exceeds guard "
                              f"{DEFAULT_DENSE_GUARD if guard is None else guard}")
    host = not isinstance(a, DeviceBta)
    A = to_device(a) if host else a
    ctx = _native.Context.get(A.device.index)
    t0 = perf_counter()
    dA = dense_device(A)
    inv = torch.empty_like(dA)
    ctx.bind_stream()
    ctx.call("bsel_block_inverse", ctypes.c_void_p(dA.data_ptr()), total, ctypes.c_void_p(inv.data_ptr()),
             total, total)
    if counter is not None:  # the reference's LU + two triangular solves
        counter.lu_count += 1
        counter.trsm_count += 2
    torch.cuda.current_stream(A.device).synchronize()
    t1 = perf_counter()
    x_a = mask_device(inv, a.shape_params)
    x_b = None
    if mode == "siq":
        B = to_device(b) if not isinstance(b, DeviceBta) else b
        dB = dense_device(B)
        y = torch.empty_like(dA)
        _gemm(ctx, y, inv, dB)
        _gemm(ctx, dB, y, inv, trans_y=True)  # reuse dB as the output
        if counter is not None:
            counter.record_gemm(total, total, total)
            counter.record_gemm(total, total, total)
        x_b = mask_device(dB, a.shape_params)
    torch.cuda.current_stream(A.device).synchronize()
    t2 = perf_counter()
    if timings is not None:
        timings["forward"] = t1 - t0
        timings["backward"] = t2 - t1
    if host:
        return SelectedSolution(x_a=to_host(x_a), x_b=to_host(x_b) if x_b is not None else None, mode=mode)
    return SelectedSolution(x_a=x_a, x_b=x_b, mode=mode)
