"""ctypes binding of the C ABI in include/btasel_b200.h (libbtasel_b200.so).

This is the thin layer between the Python facade and the sm_100a library.
It owns one ``bsel_context`` per CUDA device, maps ABI status codes to the
reference's exceptions, and never falls back to a CPU implementation: a
missing library or GPU raises NativeUnavailableError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeUnavailableError, ShapeMismatchError, SingularBlockError

LIB_NAME = "libbtasel_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

OK, ERR_SHAPE, ERR_SINGULAR, ERR_CUDA, ERR_ARG, ERR_INTERNAL = range(6)

# Every symbol include/btasel_b200.h declares (checked by tests/test_abi_exports.py).
EXPORTS = (
    "bsel_abi_version",
    "bsel_context_create",
    "bsel_context_destroy",
    "bsel_context_set_stream",
    "bsel_context_set_inverse_grid",
    "bsel_context_set_b_symmetry",
    "bsel_context_b_symmetry",
    "bsel_context_set_aux_avoid_sms",
    "bsel_synchronize",
    "bsel_last_timings",
    "bsel_block_multiply_acc",
    "bsel_block_inverse",
    "bsel_bta_forward",
    "bsel_bta_backward",
    "bsel_solve_workspace_size",
    "bsel_solve_selected",
    "bsel_local_forward",
    "bsel_local_backward",
    "bsel_generate_dd_bta",
    "bsel_hermitianize",
    "bsel_publish",
    "bsel_kernel_launches",
    "bsel_profile_begin",
    "bsel_profile_end",
)


class Status(ctypes.Structure):
    _fields_ = [
        ("code", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("index", ctypes.c_int64),
        ("message", ctypes.c_char * 256),
    ]


class Bta(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("b", ctypes.c_int64),
        ("a", ctypes.c_int64),
        ("diag", ctypes.c_void_p),
        ("lower", ctypes.c_void_p),
        ("upper", ctypes.c_void_p),
        ("arrow_row", ctypes.c_void_p),
        ("arrow_col", ctypes.c_void_p),
        ("tip", ctypes.c_void_p),
    ]


class Factors(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("b", ctypes.c_int64),
        ("a", ctypes.c_int64),
        ("fused", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("s_a", ctypes.c_void_p),
        ("s_b", ctypes.c_void_p),
        ("b_diag_last", ctypes.c_void_p),
        ("tip_inv", ctypes.c_void_p),
        ("b_tip", ctypes.c_void_p),
        ("arrow_row_elim", ctypes.c_void_p),
        ("arrow_col_elim", ctypes.c_void_p),
        ("b_arrow_row_elim", ctypes.c_void_p),
        ("b_arrow_col_elim", ctypes.c_void_p),
        ("elim_f", ctypes.c_void_p),
        ("elim_g", ctypes.c_void_p),
        ("elim_q", ctypes.c_void_p),
        ("elim_k", ctypes.c_void_p),
        ("elim_h", ctypes.c_void_p),
        ("elim_ha", ctypes.c_void_p),
        ("elim_eq", ctypes.c_void_p),
        ("elim_ek", ctypes.c_void_p),
    ]


class HostIo(ctypes.Structure):
    """bsel_host_io_t: host matrices streamed behind the partition sweeps."""

    _fields_ = [
        ("a", ctypes.POINTER(Bta)),
        ("b", ctypes.POINTER(Bta)),
        ("x_a", ctypes.POINTER(Bta)),
        ("x_b", ctypes.POINTER(Bta)),
        ("chunk_blocks", ctypes.c_int64),
        ("copy_tip", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("copy_stream", ctypes.c_void_p),
    ]


def host_desc(m) -> Bta:
    """bsel_bta_t over a host BtaMatrix's stacked (C-contiguous) arrays."""
    d = Bta()
    d.n, d.b, d.a = m.n, m.b, m.a
    for k, arr in m.stacked().items():
        if arr.size and not arr.flags["C_CONTIGUOUS"]:
            raise ValueError(f"host {k} array must be C-contiguous")
        setattr(d, k, arr.ctypes.data if arr.size else None)
    return d


class LocalFactors(ctypes.Structure):
    _fields_ = [
        ("lo", ctypes.c_int64),
        ("hi", ctypes.c_int64),
        ("kind", ctypes.c_int32),
        ("fused", ctypes.c_int32),
        ("s_a", ctypes.c_void_p),
        ("s_b", ctypes.c_void_p),
        ("fill_row", ctypes.c_void_p),
        ("fill_col", ctypes.c_void_p),
        ("b_fill_row", ctypes.c_void_p),
        ("b_fill_col", ctypes.c_void_p),
        ("elim_f", ctypes.c_void_p),
        ("elim_g", ctypes.c_void_p),
        ("elim_q", ctypes.c_void_p),
        ("elim_k", ctypes.c_void_p),
        ("elim_fr", ctypes.c_void_p),
        ("elim_qr", ctypes.c_void_p),
        ("elim_h", ctypes.c_void_p),
        ("elim_ha", ctypes.c_void_p),
        ("elim_eq", ctypes.c_void_p),
        ("elim_ek", ctypes.c_void_p),
    ]


class Profile(ctypes.Structure):
    _fields_ = [
        ("gemm_launches", ctypes.c_int64),
        ("gemm_flops", ctypes.c_double),
        ("gemm_ms", ctypes.c_double),
        ("inverse_calls", ctypes.c_int64),
        ("inverse_ms", ctypes.c_double),
        ("gemm_bytes", ctypes.c_double),
        ("gemm_busy_ms", ctypes.c_double),
        ("inverse_busy_ms", ctypes.c_double),
        ("inverse_flops", ctypes.c_double),
        ("gemm_exec_flops", ctypes.c_double),
    ]


_lib = None
_lock = threading.Lock()


def load_library(path: str | None = None) -> ctypes.CDLL:
    """Load (once) and type the C ABI.  Does not need a GPU."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or LIB_PATH
        if not os.path.exists(p):
            raise NativeUnavailableError(
                f"{LIB_NAME} not found at {p}: run __graft_entry__.build() (make -C "
                "paper_2601_04904_b200/csrc); there is no CPU fallback"
            )
        lib = ctypes.CDLL(p)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        st = ctypes.POINTER(Status)
        sig = {
            "bsel_abi_version": ([], i32),
            "bsel_context_create": ([i32, ctypes.POINTER(vp), st], i32),
            "bsel_context_destroy": ([vp], i32),
            "bsel_context_set_stream": ([vp, vp], i32),
            "bsel_context_set_inverse_grid": ([vp, i32], i32),
            "bsel_context_set_b_symmetry": ([vp, i32], i32),
            "bsel_context_b_symmetry": ([vp, ctypes.POINTER(i32), ctypes.POINTER(i32)], i32),
            "bsel_context_set_aux_avoid_sms": ([vp, i32], i32),
            "bsel_synchronize": ([vp, st], i32),
            "bsel_last_timings": ([vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], i32),
            "bsel_block_multiply_acc": (
                [vp, vp, i64, vp, i64, vp, i64, i32, vp, i64, i32, i64, i64, i64,
                 ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double, st], i32),
            "bsel_block_inverse": ([vp, vp, i64, vp, i64, i64, st], i32),
            "bsel_bta_forward": ([vp, ctypes.POINTER(Bta), ctypes.POINTER(Bta), ctypes.POINTER(Factors), st], i32),
            "bsel_bta_backward": ([vp, ctypes.POINTER(Factors), ctypes.POINTER(Bta), ctypes.POINTER(Bta),
                                   ctypes.POINTER(Bta), ctypes.POINTER(Bta), i32, st], i32),
            "bsel_solve_workspace_size": ([i64, i64, i64, i32, ctypes.POINTER(ctypes.c_size_t)], i32),
            "bsel_solve_selected": ([vp, ctypes.POINTER(Bta), ctypes.POINTER(Bta), ctypes.POINTER(Bta),
                                     ctypes.POINTER(Bta), i32, vp, ctypes.c_size_t, st], i32),
        }
        lf = ctypes.POINTER(LocalFactors)
        pb = ctypes.POINTER(Bta)
        ts = ctypes.POINTER(HostIo)
        sig["bsel_local_forward"] = ([vp, pb, pb, pb, pb, lf, ts, st], i32)
        sig["bsel_local_backward"] = ([vp, pb, pb, lf, pb, pb, pb, pb, i64, i64, i32, pb, pb, ts, st], i32)
        sig["bsel_generate_dd_bta"] = ([vp, ctypes.POINTER(Bta), ctypes.c_uint64, ctypes.c_double, st], i32)
        sig["bsel_hermitianize"] = ([vp, ctypes.POINTER(Bta), st], i32)
        sig["bsel_publish"] = ([vp, vp, vp, vp, i32, vp, i32, i64, vp, st], i32)
        sig["bsel_kernel_launches"] = ([], ctypes.c_uint64)
        sig["bsel_profile_begin"] = ([], i32)
        sig["bsel_profile_end"] = ([ctypes.POINTER(Profile)], i32)
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        if lib.bsel_abi_version() != 3:
            raise NativeUnavailableError("ABI version mismatch")
        if path is None:
            _lib = lib
        return lib


def raise_for_status(code: int, st: Status) -> None:
    if code == OK:
        return
    msg = st.message.decode(errors="replace")
    if code == ERR_SINGULAR:
        raise SingularBlockError(msg, index=int(st.index))
    if code == ERR_SHAPE:
        raise ShapeMismatchError(msg)
    if code == ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"btasel_b200 native error {code}: {msg}")


class Context:
    """A bsel_context per (device, lane); calls run on torch's current stream.

    Lane 0 is the default.  Extra lanes (own streams, slot pools and
    inverse workspaces inside the native context) let independent partitions
    of the distributed scheme run concurrently on one GPU from separate
    Python threads (ctypes releases the GIL during native calls).
    """

    _per_device: dict = {}
    _lock = threading.Lock()

    def __init__(self, device: int):
        self.lib = load_library()
        self.device = device
        handle = ctypes.c_void_p()
        st = Status()
        raise_for_status(self.lib.bsel_context_create(device, ctypes.byref(handle), ctypes.byref(st)), st)
        self.handle = handle

    @classmethod
    def get(cls, device: int | None = None, lane: int = 0) -> "Context":
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailableError("no CUDA device: the B200 solver has no CPU fallback")
        if device is None:
            device = torch.cuda.current_device()
        with cls._lock:
            ctx = cls._per_device.get((device, lane))
            if ctx is None:
                with torch.cuda.device(device):
                    ctx = cls(device)
                cls._per_device[(device, lane)] = ctx
        ctx.bind_stream()
        return ctx

    def bind_stream(self, stream=None) -> None:
        import torch

        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.lib.bsel_context_set_stream(self.handle, ctypes.c_void_p(s.cuda_stream))

    def set_inverse_grid(self, ctas: int) -> None:
        """CTAs of the persistent block inverse on this context (0 = default)."""
        if self.lib.bsel_context_set_inverse_grid(self.handle, int(ctas)) != 0:
            raise ValueError(f"invalid inverse grid {ctas}")

    SYM_AUTO = 2

    def set_b_symmetry(self, mode: int) -> None:
        """Backward path for the quadratic solve: +1 / -1 (B = +-B^H), 0
        (general) or SYM_AUTO (this context's own check of B)."""
        if self.lib.bsel_context_set_b_symmetry(self.handle, int(mode)) != 0:
            raise ValueError(f"invalid symmetry mode {mode}")

    def set_aux_avoid_sms(self, n: int) -> None:
        """Forward aux GEMM levels leave SMs [0, n) to the chain (0 = off)."""
        if self.lib.bsel_context_set_aux_avoid_sms(self.handle, int(n)) != 0:
            raise ValueError(f"invalid SM count {n}")

    def b_symmetry(self) -> tuple[int, int]:
        """(flags of the last check of B, path the backward would take)."""
        flags, mode = ctypes.c_int32(), ctypes.c_int32()
        self.lib.bsel_context_b_symmetry(self.handle, ctypes.byref(flags), ctypes.byref(mode))
        return flags.value, mode.value

    def call(self, name: str, *args) -> None:
        st = Status()
        code = getattr(self.lib, name)(self.handle, *args, ctypes.byref(st))
        raise_for_status(code, st)

    def timings(self) -> tuple[float, float]:
        f, b = ctypes.c_double(), ctypes.c_double()
        self.lib.bsel_last_timings(self.handle, ctypes.byref(f), ctypes.byref(b))
        return f.value, b.value

    def workspace_bytes(self, n: int, b: int, a: int, fused: bool) -> int:
        out = ctypes.c_size_t()
        self.lib.bsel_solve_workspace_size(n, b, a, int(fused), ctypes.byref(out))
        return out.value
