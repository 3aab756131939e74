"""Sequential selected inversion / fused selected quadratic solution on the
B200 (drop-in for btasel/rgf.py).

The forward Schur sweep, the fused SI+SQ backward sweep, the per-block
inverse and the arrowhead tip update all run inside libbtasel_b200.so
(csrc/sweeps.cu) as stream-ordered grouped DMMA GEMM levels; this module
only marshals containers across the C ABI:

* host ``BtaMatrix`` in  -> host ``BtaMatrix`` out (reference semantics,
  one memcpy per block kind each way);
* ``DeviceBta`` in -> ``DeviceBta`` out (zero-copy fast path).

Entry points and semantics follow the reference (rgf.py:79, 127, 207, 401,
497): ``*_forward`` mutate their working copies in place and return
``RgfFactors``; ``solve_selected`` never mutates its inputs.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native
from .device import DeviceBta
from .errors import ShapeMismatchError
from .kernels import OpCounter, record_sweep
from .matrix import BtaMatrix, SelectedSolution

__all__ = ["RgfFactors", "bt_forward", "bt_backward", "bta_forward", "bta_backward", "solve_selected"]


@dataclass
class RgfFactors:
    """Schur data retained between the sweeps (rgf.py:37-61).

    Host-visible fields mirror the reference (lists of blocks).  ``_dev``
    keeps the device-resident copy produced by the forward sweep so that a
    following backward sweep does not re-upload it.
    """

    n: int
    b: int
    a: int
    mode: str
    s_a: list = field(default_factory=list)
    s_b: list | None = None
    b_diag_last: np.ndarray | None = None
    arrow_row_elim: list | None = None
    arrow_col_elim: list | None = None
    b_arrow_row_elim: list | None = None
    b_arrow_col_elim: list | None = None
    tip_schur_inv: np.ndarray | None = None
    b_tip: np.ndarray | None = None
    _dev: dict | None = field(default=None, repr=False)


def _check_mode(a, b, mode):
    if mode is None:
        mode = "si" if b is None else "siq"
    if mode not in ("si", "siq"):
        raise ValueError(f"mode must be 'si' or 'siq', got {mode!r}")
    if mode == "siq" and b is None:
        raise ValueError("mode 'siq' requires a right-hand side")
    return mode


def _ctx_for(x, pipe=0):
    """Native context of the device holding x (the current device for host
    inputs); ``pipe`` > 0 (concurrent solves of EnergySweep) selects a lane
    of its own."""
    dev = x.device.index if isinstance(x, DeviceBta) else None
    ctx = _native.Context.get(dev, lane=0 if pipe == 0 else 1000 + pipe)
    return ctx, torch.device("cuda", ctx.device)


def _ptr(t):
    return t.data_ptr() if (t is not None and t.numel()) else None


def _factor_desc(n, b, a, fused, dev: dict, A: DeviceBta, B: DeviceBta | None) -> _native.Factors:
    f = _native.Factors()
    f.n, f.b, f.a, f.fused = n, b, a, int(fused)
    f.s_a = _ptr(dev["s_a"])
    f.tip_inv = _ptr(dev["tip_inv"])
    f.arrow_row_elim = _ptr(A.arrow_row)
    f.arrow_col_elim = _ptr(A.arrow_col)
    if fused:
        f.s_b = _ptr(dev["s_b"])
        f.b_diag_last = _ptr(dev["b_diag_last"])
        f.b_tip = _ptr(dev["b_tip"])
        f.b_arrow_row_elim = _ptr(B.arrow_row)
        f.b_arrow_col_elim = _ptr(B.arrow_col)
    for k in _ELIM:
        setattr(f, k, _ptr(dev.get(k)))
    return f


_ELIM = ("elim_f", "elim_g", "elim_q", "elim_k", "elim_h", "elim_ha", "elim_eq", "elim_ek")


def _alloc_elim(n, b, a, fused, c128) -> dict:
    """Elimination products retained forward -> backward (bsel_factors_t),
    the same set bsel_solve_selected keeps, so the split forward / backward
    runs exactly the facade's kernels (bitwise equal results, reference
    acceptance criterion 8, test_acceptance.py:290-305)."""
    import os

    extra = os.environ.get("BSEL_FWD_BWD_PRODUCTS", "0") not in ("", "0")
    e = {"elim_f": torch.empty((n, b, b), **c128), "elim_h": torch.empty((n, b, b), **c128)}
    if a:
        e["elim_g"] = torch.empty((n, a, b), **c128)
        if extra or not fused:
            e["elim_ha"] = torch.empty((n, b, a), **c128)
    if fused:
        e["elim_q"] = torch.empty((n, b, b), **c128)
        if a:
            e["elim_k"] = torch.empty((n, b, a), **c128)
        if extra:
            e["elim_eq"] = torch.empty((n, b, b), **c128)
            if a:
                e["elim_ek"] = torch.empty((n, b, a), **c128)
    return e


def _forward(a, b, counter, require_bt):
    if require_bt and a.a != 0:
        raise ShapeMismatchError("bt_forward requires a plain BT matrix (a=0)")
    if b is not None and b.shape_params != a.shape_params:
        raise ShapeMismatchError("right-hand side shape differs from system shape")
    n, bs, asz = a.shape_params
    fused = b is not None
    ctx, device = _ctx_for(a)
    host = not isinstance(a, DeviceBta)
    A = DeviceBta.empty(n, bs, asz, device, zero=False).copy_from_host(a) if host else a
    B = None
    if fused:
        B = DeviceBta.empty(n, bs, asz, device, zero=False).copy_from_host(b) if host else b
    c128 = dict(dtype=torch.complex128, device=device)
    dev = {"s_a": torch.empty((n, bs, bs), **c128), "tip_inv": torch.empty((asz, asz), **c128)}
    if fused:
        dev.update(s_b=torch.empty((max(n - 1, 0), bs, bs), **c128),
                   b_diag_last=torch.empty((bs, bs), **c128), b_tip=torch.empty((asz, asz), **c128))
    dev.update(_alloc_elim(n, bs, asz, fused, c128))
    fd = _factor_desc(n, bs, asz, fused, dev, A, B)
    ad = A.desc()
    bd = B.desc() if fused else None
    ctx.bind_stream()
    ctx.call("bsel_bta_forward", ctypes.byref(ad), ctypes.byref(bd) if fused else None, ctypes.byref(fd))
    record_sweep(counter, n, bs, asz, "siq" if fused else "si", "forward")
    dev["A"], dev["B"] = A, B
    fac = RgfFactors(n=n, b=bs, a=asz, mode="siq" if fused else "si", _dev=dev)
    if host:
        # Reference semantics: the working copies are updated in place and the
        # factor lists alias them (rgf.py:84-86, 240-244).
        A.copy_to_host(a)
        if fused:
            B.copy_to_host(b)
        s_a = dev["s_a"].cpu().numpy()
        fac.s_a = [s_a[i] for i in range(n)]
        if asz:
            fac.arrow_row_elim = list(a.arrow_row)
            fac.arrow_col_elim = list(a.arrow_col)
            fac.tip_schur_inv = dev["tip_inv"].cpu().numpy()
        if fused:
            s_b = dev["s_b"].cpu().numpy()
            fac.s_b = [s_b[i] for i in range(n - 1)]
            fac.b_diag_last = dev["b_diag_last"].cpu().numpy()
            if asz:
                fac.b_arrow_row_elim = list(b.arrow_row)
                fac.b_arrow_col_elim = list(b.arrow_col)
                fac.b_tip = dev["b_tip"].cpu().numpy()
    else:
        fac.s_a = list(dev["s_a"])
        fac.tip_schur_inv = dev["tip_inv"] if asz else None
        if asz:
            fac.arrow_row_elim, fac.arrow_col_elim = list(A.arrow_row), list(A.arrow_col)
        if fused:
            fac.s_b = list(dev["s_b"])
            fac.b_diag_last = dev["b_diag_last"]
            if asz:
                fac.b_tip = dev["b_tip"]
                fac.b_arrow_row_elim, fac.b_arrow_col_elim = list(B.arrow_row), list(B.arrow_col)
    return fac


def _upload_factors(f: RgfFactors, device):
    """Rebuild device factors from host lists (backward without a device forward)."""
    n, bs, asz = f.n, f.b, f.a
    fused = f.mode == "siq"
    t = lambda x, shape: (torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.complex128)).reshape(shape))  # noqa: E731
                          .to(device))
    dev = {"s_a": t(np.stack(f.s_a), (n, bs, bs)),
           "tip_inv": t(f.tip_schur_inv if asz else np.zeros((0, 0)), (asz, asz))}
    A = DeviceBta.empty(n, bs, asz, device)
    if asz:
        A.arrow_row.copy_(t(np.stack(f.arrow_row_elim), (n, asz, bs)))
        A.arrow_col.copy_(t(np.stack(f.arrow_col_elim), (n, bs, asz)))
    B = None
    if fused:
        dev["s_b"] = t(np.stack(f.s_b) if n > 1 else np.zeros((0, bs, bs)), (n - 1, bs, bs))
        dev["b_diag_last"] = t(f.b_diag_last, (bs, bs))
        dev["b_tip"] = t(f.b_tip if asz else np.zeros((0, 0)), (asz, asz))
        B = DeviceBta.empty(n, bs, asz, device)
        if asz:
            B.arrow_row.copy_(t(np.stack(f.b_arrow_row_elim), (n, asz, bs)))
            B.arrow_col.copy_(t(np.stack(f.b_arrow_col_elim), (n, bs, asz)))
    dev["A"], dev["B"] = A, B
    return dev


def _backward(factors: RgfFactors, a, b, counter, diagonal_only, require_bt):
    n, bs, asz = factors.n, factors.b, factors.a
    if require_bt and asz != 0:
        raise ShapeMismatchError("bt_backward requires BT factors (a=0)")
    if a.shape_params != (n, bs, asz):
        raise ShapeMismatchError("system shape disagrees with factors")
    fused = factors.mode == "siq"
    if fused and b is None:
        raise ShapeMismatchError("fused factors require the right-hand side")
    ctx, device = _ctx_for(a)
    host = not isinstance(a, DeviceBta)
    dev = factors._dev if factors._dev is not None else _upload_factors(factors, device)
    A_off = DeviceBta.empty(n, bs, asz, device, zero=False) if host else a
    if host:
        A_off.lower.copy_(torch.from_numpy(a.stacked()["lower"]))
        A_off.upper.copy_(torch.from_numpy(a.stacked()["upper"]))
    B_off = None
    if fused:
        B_off = DeviceBta.empty(n, bs, asz, device, zero=False) if host else b
        if host:
            B_off.lower.copy_(torch.from_numpy(b.stacked()["lower"]))
            B_off.upper.copy_(torch.from_numpy(b.stacked()["upper"]))
    XA = DeviceBta.empty(n, bs, asz, device)
    XB = DeviceBta.empty(n, bs, asz, device) if fused else None
    fd = _factor_desc(n, bs, asz, fused, dev, dev["A"], dev["B"])
    ad, xad = A_off.desc(), XA.desc()
    bd = B_off.desc() if fused else None
    xbd = XB.desc() if fused else None
    ctx.bind_stream()
    ctx.call("bsel_bta_backward", ctypes.byref(fd), ctypes.byref(ad), ctypes.byref(bd) if fused else None,
             ctypes.byref(xad), ctypes.byref(xbd) if fused else None, int(bool(diagonal_only)))
    record_sweep(counter, n, bs, asz, factors.mode, "backward")
    if host:
        from .device import to_host

        return SelectedSolution(x_a=to_host(XA), x_b=to_host(XB) if fused else None, mode=factors.mode)
    return SelectedSolution(x_a=XA, x_b=XB, mode=factors.mode)


def bt_forward(a, b=None, counter: OpCounter | None = None) -> RgfFactors:
    """Forward Schur pass over a BT system (rgf.py:79-124, Alg. 1)."""
    return _forward(a, b, counter, require_bt=True)


def bt_backward(factors, a, b=None, counter=None, *, diagonal_only=False) -> SelectedSolution:
    """Backward selected substitution over a BT system (rgf.py:127-199, Alg. 2)."""
    return _backward(factors, a, b, counter, diagonal_only, require_bt=True)


def bta_forward(a, b=None, counter: OpCounter | None = None) -> RgfFactors:
    """Forward pass over an arrowhead system (rgf.py:207-319); a=0 -> BT."""
    return _forward(a, b, counter, require_bt=False)


def bta_backward(factors, a, b=None, counter=None, *, diagonal_only=False) -> SelectedSolution:
    """Backward pass over an arrowhead system (rgf.py:401-489); a=0 -> BT."""
    return _backward(factors, a, b, counter, diagonal_only, require_bt=False)


_PARTITIONED = {}


def _pinned(m) -> bool:
    """True when every array of host BtaMatrix ``m`` is page-locked."""
    return all(torch.from_numpy(x).is_pinned() for x in m.stacked().values() if x.size)


def default_partitions(n: int) -> int:
    """Partitions used by ``solve_selected(partitions=None)``: the 2-partition
    scheme run concurrently on one GPU once the chain is long enough to
    matter (config 4: 784 vs 978 ms per energy point); BSEL_PARTITIONS
    overrides (1 = always the sequential RGF sweeps)."""
    import os

    env = os.environ.get("BSEL_PARTITIONS")
    if env:
        return max(1, int(env))
    return 2 if n >= 64 else 1


def release_caches() -> None:
    """Drop cached partition buffers of ``solve_selected(partitions>1)``."""
    _PARTITIONED.clear()


def solve_selected(a, b=None, mode=None, *, counter=None, timings=None, diagonal_only=False,
                   out=None, workspace=None, partitions=None, _b_symmetry=None, _device_in=None,
                   _io_events=None, _pipe=0, _device_out=None) -> SelectedSolution:
    """Selected inverse of ``a`` and, in fused mode, the selected quadratic
    solution for ``b`` (rgf.py:497-531).  Never mutates its inputs.

    Host ``BtaMatrix`` inputs return host containers; ``DeviceBta`` inputs
    stay on the GPU.  ``out`` may pass preallocated (x_a, x_b): DeviceBta
    (device outputs) or host BtaMatrix (e.g. pinned, filled by async D2H);
    ``timings`` receives the device-timed forward/backward seconds.

    ``partitions``: 1 = the sequential RGF sweeps (rgf.py); k > 1 = the
    paper's partitioned scheme (dist.py) with all k partitions running
    concurrently on this GPU; None = ``default_partitions(n)``.  Both agree
    with the reference to ~1e-15; ``counter`` always receives the reference's
    sequential inventory.
    """
    mode = _check_mode(a, b, mode)
    fused = mode == "siq"
    if fused and b.shape_params != a.shape_params:
        raise ShapeMismatchError("right-hand side shape differs from system shape")
    n, bs, asz = a.shape_params
    parts = default_partitions(n) if partitions is None else int(partitions)
    if parts > 1 and n >= 2 * parts:
        return _solve_partitioned(a, b if fused else None, mode, parts, counter, timings, diagonal_only, out,
                                  _device_in, _io_events, _pipe, _device_out)
    ctx, device = _ctx_for(a, _pipe)
    host = not isinstance(a, DeviceBta)
    A = DeviceBta.empty(n, bs, asz, device, zero=False).copy_from_host(a) if host else a
    B = None
    if fused:
        B = DeviceBta.empty(n, bs, asz, device, zero=False).copy_from_host(b) if host else b
    host_out = None
    if out is not None and isinstance(out[0], DeviceBta):
        XA, XB = out
        if diagonal_only:
            XA.lower.zero_()
            XA.upper.zero_()
            if XB is not None:
                XB.lower.zero_()
                XB.upper.zero_()
    else:
        # host outputs (optionally caller-provided, e.g. pinned BtaMatrix.zeros(pinned=True))
        host_out = out
        XA = DeviceBta.empty(n, bs, asz, device, zero=diagonal_only or out is None)
        XB = DeviceBta.empty(n, bs, asz, device, zero=diagonal_only or out is None) if fused else None
    need = ctx.workspace_bytes(n, bs, asz, fused)
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=device)
    ad, xad = A.desc(), XA.desc()
    bd = B.desc() if fused else None
    xbd = XB.desc() if fused else None
    ctx.bind_stream()
    # _b_symmetry (internal): the partitioned solves force the backward path
    # decided for the whole B; by default the solve uses its own check of B.
    if _b_symmetry is not None:
        ctx.set_b_symmetry(_b_symmetry)
    try:
        ctx.call("bsel_solve_selected", ctypes.byref(ad), ctypes.byref(bd) if fused else None, ctypes.byref(xad),
                 ctypes.byref(xbd) if fused else None, int(bool(diagonal_only)),
                 ctypes.c_void_p(workspace.data_ptr()), workspace.numel())
    finally:
        if _b_symmetry is not None:
            ctx.set_b_symmetry(ctx.SYM_AUTO)
    record_sweep(counter, n, bs, asz, mode, "forward")
    record_sweep(counter, n, bs, asz, mode, "backward")
    if timings is not None:
        fwd_ms, bwd_ms = ctx.timings()
        timings["forward"] = fwd_ms / 1e3
        timings["backward"] = bwd_ms / 1e3
    if host_out is not None:
        hxa, hxb = host_out
        XA.copy_to_host(hxa, non_blocking=True)
        if fused:
            XB.copy_to_host(hxb, non_blocking=True)
        torch.cuda.current_stream(device).synchronize()
        return SelectedSolution(x_a=hxa, x_b=hxb if fused else None, mode=mode)
    if host and not (out is not None and isinstance(out[0], DeviceBta)):
        from .device import to_host

        return SelectedSolution(x_a=to_host(XA), x_b=to_host(XB) if fused else None, mode=mode)
    # device outputs given by the caller stay on the device (host inputs or not)
    return SelectedSolution(x_a=XA, x_b=XB, mode=mode)


def _solve_partitioned(a, b, mode, parts, counter, timings, diagonal_only, out, device_in=None, io_events=None,
                       pipe=0, device_out=None):
    """solve_selected through InGpuPartitions (dist.py) with cached buffers.

    ``device_in`` (internal, HostEnergySweep): device storage for streamed
    host inputs instead of a fresh allocation; ``io_events`` receives
    "inputs_done", the event after the last streamed input chunk;
    ``device_out``: device storage behind streamed host outputs."""
    from .dist import InGpuPartitions

    n, bs, asz = a.shape_params
    fused = b is not None
    _, device = _ctx_for(a)
    host = not isinstance(a, DeviceBta)
    # Pinned host inputs are streamed in behind the forward sweeps and pinned
    # host outputs out behind the backward sweeps (bsel_host_io_t); pageable
    # memory would make every chunk copy synchronous, so it is moved whole.
    stream_in = host and _pinned(a) and (b is None or _pinned(b))
    host_out = out if (out is not None and not isinstance(out[0], DeviceBta)) else None
    stream_out = host_out is not None and not diagonal_only and all(_pinned(x) for x in host_out if x is not None)
    dev_in = device_in if (host and device_in is not None) else None
    A = a if not host else (dev_in[0] if dev_in else DeviceBta.empty(n, bs, asz, device, zero=False))
    if host and not stream_in:
        A.copy_from_host(a)
    B = None
    if fused:
        B = b if not host else (dev_in[1] if dev_in else DeviceBta.empty(n, bs, asz, device, zero=False))
        if host and not stream_in:
            B.copy_from_host(b)
    # pipe (internal, EnergySweep concurrency): concurrent solves need their own
    # runner (factor buffers) and lane contexts
    key = (device.index, n, bs, asz, mode, parts, pipe)
    runner = _PARTITIONED.get(key)
    if runner is None:
        runner = _PARTITIONED[key] = InGpuPartitions((n, bs, asz), mode, parts, device, lane_base=pipe * parts,
                                                     pipe=pipe)
    dev_out = out if (out is not None and isinstance(out[0], DeviceBta)) else None
    if dev_out is None and stream_out and device_out is not None:
        dev_out = device_out
    if stream_in or stream_out:
        XA, XB = runner.run(A, B, out=dev_out, host_in=(a, b) if stream_in else None,
                            host_out=host_out if stream_out else None)
    else:
        XA, XB = runner.run(A, B, out=dev_out)
    if io_events is not None and stream_in:
        ev = torch.cuda.Event()
        ev.record(runner.copy_stream)
        io_events["inputs_done"] = ev
        cb = io_events.get("on_inputs_done")
        if cb is not None:  # before the host-output synchronization below
            cb(ev)
    if stream_out:
        record_sweep(counter, n, bs, asz, mode, "forward")
        record_sweep(counter, n, bs, asz, mode, "backward")
        if timings is not None:
            ph = runner.phase_seconds()
            timings["forward"] = ph["forward"] + ph["communication"] + ph["reduced"]
            timings["backward"] = ph["backward"]
        torch.cuda.current_stream(device).synchronize()
        return SelectedSolution(x_a=host_out[0], x_b=host_out[1] if fused else None, mode=mode,
                                algorithm=f"partitions={parts}")
    if diagonal_only:
        for X in (XA, XB) if fused else (XA,):
            X.lower.zero_()
            X.upper.zero_()
    record_sweep(counter, n, bs, asz, mode, "forward")
    record_sweep(counter, n, bs, asz, mode, "backward")
    if timings is not None:
        ph = runner.phase_seconds()
        timings["forward"] = ph["forward"] + ph["communication"] + ph["reduced"]
        timings["backward"] = ph["backward"]
    if out is not None and not isinstance(out[0], DeviceBta):
        hxa, hxb = out
        XA.copy_to_host(hxa, non_blocking=True)
        if fused:
            XB.copy_to_host(hxb, non_blocking=True)
        torch.cuda.current_stream(device).synchronize()
        return SelectedSolution(x_a=hxa, x_b=hxb if fused else None, mode=mode, algorithm=f"partitions={parts}")
    if host and dev_out is None:
        from .device import to_host

        return SelectedSolution(x_a=to_host(XA), x_b=to_host(XB) if fused else None, mode=mode,
                                algorithm=f"partitions={parts}")
    # device outputs given by the caller stay on the device (host inputs or not): a
    # round-1 bug copied them to pageable host memory here (the "8.5 s streamed first
    # energy" of HostEnergySweep with two output slots)
    return SelectedSolution(x_a=XA, x_b=XB, mode=mode, algorithm=f"partitions={parts}")
