"""BT(A) containers with stacked, transfer-ready storage (mirrors btasel/matrix.py).

The reference stores a BtaMatrix as Python lists of blocks
(matrix.py:35-72).  Here every block kind lives in ONE contiguous
``[count, rows, cols]`` complex128 array -- the exact byte layout of the C
ABI (include/btasel_b200.h) and of the BTA1 payload -- so a host <-> device
transfer is a single memcpy per kind and can come from pinned memory.  The
list API of the reference is preserved through :class:`BlockList` views:
``m.diag[i]`` is a writable view into the stack and ``m.diag[i] = x``
copies ``x`` into place.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ShapeMismatchError

COMPLEX = np.complex128
KINDS = ("diag", "lower", "upper", "arrow_row", "arrow_col")
MODES = ("si", "siq")

__all__ = [
    "BtaMatrix",
    "BlockList",
    "SelectedSolution",
    "generate_dd_bta",
    "to_dense",
    "mask_to_pattern",
    "hermitianize",
]


class BlockList:
    """List-like view over a stacked ``[count, r, c]`` array."""

    __slots__ = ("_stack",)

    def __init__(self, stack: np.ndarray):
        self._stack = stack

    def __len__(self):
        return self._stack.shape[0]

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._stack[j] for j in range(*i.indices(len(self)))]
        return self._stack[i]

    def __setitem__(self, i, value):
        value = np.asarray(value, dtype=COMPLEX)
        if value.shape != self._stack.shape[1:]:
            raise ShapeMismatchError(f"block has shape {value.shape}, expected {self._stack.shape[1:]}")
        self._stack[i] = value

    def __iter__(self):
        return (self._stack[j] for j in range(len(self)))

    def __repr__(self):
        return f"BlockList({len(self)} x {self._stack.shape[1:]})"


def _stack_blocks(blocks, count, shape, name, alloc):
    out = alloc((count,) + shape)
    if isinstance(blocks, np.ndarray) and blocks.ndim == 3:
        if blocks.shape != (count,) + shape:
            raise ShapeMismatchError(f"{name} has shape {blocks.shape}, expected {(count,) + shape}")
        out[...] = blocks
        return out
    blocks = list(blocks)
    if len(blocks) != count:
        raise ShapeMismatchError(f"{name} has {len(blocks)} blocks, expected {count}")
    for i, blk in enumerate(blocks):
        arr = np.asarray(blk, dtype=COMPLEX)
        if arr.shape != shape:
            raise ShapeMismatchError(f"{name}[{i}] has shape {arr.shape}, expected {shape}")
        out[i] = arr
    return out


def _numpy_alloc(shape):
    return np.zeros(shape, dtype=COMPLEX)


def pinned_alloc(shape, zero=True):
    """Page-locked host allocation (fast, async-capable H2D/D2H)."""
    import torch

    mk = torch.zeros if zero else torch.empty
    t = mk(shape, dtype=torch.complex128, pin_memory=torch.cuda.is_available())
    return t.numpy()


class BtaMatrix:
    """Pattern blocks of a BT(A) matrix (reference matrix.py:35-163).

    ``n`` diagonal blocks of size ``b``; ``lower[i]`` = block (i+1, i),
    ``upper[i]`` = block (i, i+1); ``arrow_row[i]`` (a x b) = block (t, i),
    ``arrow_col[i]`` (b x a) = block (i, t); ``tip`` (a x a).  a = 0 is BT.
    Block arguments may be lists of blocks or stacked 3-d arrays.
    """

    def __init__(self, n, b, a, diag, lower, upper, arrow_row=None, arrow_col=None, tip=None, *,
                 alloc=None):
        if n < 1 or b < 1 or a < 0:
            raise ShapeMismatchError(f"invalid shape parameters (n={n}, b={b}, a={a})")
        self.n, self.b, self.a = int(n), int(b), int(a)
        n, b, a = self.n, self.b, self.a
        alloc = alloc or _numpy_alloc
        self._diag = _stack_blocks(diag, n, (b, b), "diag", alloc)
        self._lower = _stack_blocks(lower, n - 1, (b, b), "lower", alloc)
        self._upper = _stack_blocks(upper, n - 1, (b, b), "upper", alloc)
        self._arrow_row = (alloc((n, a, b)) if arrow_row is None
                           else _stack_blocks(arrow_row, n, (a, b), "arrow_row", alloc))
        self._arrow_col = (alloc((n, b, a)) if arrow_col is None
                           else _stack_blocks(arrow_col, n, (b, a), "arrow_col", alloc))
        self._tip = alloc((a, a))
        if tip is not None:
            t = np.asarray(tip, dtype=COMPLEX)
            if t.shape != (a, a):
                raise ShapeMismatchError(f"tip has shape {t.shape}, expected {(a, a)}")
            self._tip[...] = t

    # -- list-style access (reference API) ---------------------------------
    def _kind(name):  # noqa: N805 - property factory
        attr = "_" + name

        def get(self):
            return BlockList(getattr(self, attr))

        def put(self, blocks):
            cur = getattr(self, attr)
            cur[...] = _stack_blocks(blocks, cur.shape[0], cur.shape[1:], name, _numpy_alloc)

        return property(get, put)

    diag = _kind("diag")
    lower = _kind("lower")
    upper = _kind("upper")
    arrow_row = _kind("arrow_row")
    arrow_col = _kind("arrow_col")
    del _kind

    @property
    def tip(self):
        return self._tip

    @tip.setter
    def tip(self, value):
        v = np.asarray(value, dtype=COMPLEX)
        if v.shape != self._tip.shape:
            raise ShapeMismatchError(f"tip has shape {v.shape}, expected {self._tip.shape}")
        self._tip[...] = v

    # -- stacked access (zero-copy, transfer layout) -------------------------
    def stacked(self) -> dict:
        return {"diag": self._diag, "lower": self._lower, "upper": self._upper,
                "arrow_row": self._arrow_row, "arrow_col": self._arrow_col, "tip": self._tip}

    @classmethod
    def from_stacked(cls, n, b, a, arrays: dict, *, copy=False) -> "BtaMatrix":
        m = cls.__new__(cls)
        m.n, m.b, m.a = int(n), int(b), int(a)
        for k in KINDS + ("tip",):
            arr = arrays[k]
            setattr(m, "_" + k, np.array(arr, dtype=COMPLEX, copy=True) if copy else arr)
        return m

    @property
    def shape_params(self):
        return (self.n, self.b, self.a)

    @property
    def total_size(self) -> int:
        return self.n * self.b + self.a

    @property
    def nbytes(self) -> int:
        return sum(x.nbytes for x in self.stacked().values())

    @classmethod
    def zeros(cls, n, b, a=0, *, pinned=False, zero=True) -> "BtaMatrix":
        """All-zero container; ``pinned`` = page-locked host memory (async
        transfers); ``zero=False`` skips the fill (pinned only)."""
        alloc = (lambda s: pinned_alloc(s, zero)) if pinned else _numpy_alloc
        m = cls.__new__(cls)
        m.n, m.b, m.a = int(n), int(b), int(a)
        m._diag, m._lower, m._upper = alloc((n, b, b)), alloc((n - 1, b, b)), alloc((n - 1, b, b))
        m._arrow_row, m._arrow_col, m._tip = alloc((n, a, b)), alloc((n, b, a)), alloc((a, a))
        return m

    @classmethod
    def identity(cls, n, b, a=0) -> "BtaMatrix":
        m = cls.zeros(n, b, a)
        idx = np.arange(b)
        m._diag[:, idx, idx] = 1.0
        m._tip[np.arange(a), np.arange(a)] = 1.0
        return m

    def copy(self, *, pinned=False) -> "BtaMatrix":
        out = BtaMatrix.zeros(self.n, self.b, self.a, pinned=pinned)
        for k, v in self.stacked().items():
            getattr(out, "_" + k)[...] = v
        return out

    def pattern_blocks(self):
        """Yield ``(kind, index, block)`` over all pattern blocks (matrix.py:141-153)."""
        for k in KINDS:
            for i, blk in enumerate(getattr(self, "_" + k)):
                yield (k, i, blk)
        yield ("tip", 0, self._tip)

    def equals_exact(self, other) -> bool:
        if self.shape_params != other.shape_params:
            return False
        return all(np.array_equal(x[2], y[2]) for x, y in zip(self.pattern_blocks(), other.pattern_blocks()))

    def __repr__(self):
        return f"BtaMatrix(n={self.n}, b={self.b}, a={self.a})"


@dataclass
class SelectedSolution:
    """Pattern-restricted solution containers (matrix.py:166-185).

    ``algorithm`` (not in the reference; informational): which scheme
    produced the solution -- "rgf" (the sequential sweeps, rgf.py) or
    "partitions=k" (the paper's partitioned scheme, dist.py, with k
    partitions: solve_selected's default for n >= 64 runs 2 of them
    concurrently on one GPU; ``partitions=1`` or BSEL_PARTITIONS=1 selects
    the sequential sweeps).  OpCounter always receives the reference's
    sequential inventory."""

    x_a: object
    x_b: object | None
    mode: str
    algorithm: str = "rgf"

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if (self.x_b is not None) != (self.mode == "siq"):
            raise ValueError("x_b must be present exactly in 'siq' mode")
        if self.x_b is not None and self.x_b.shape_params != self.x_a.shape_params:
            raise ShapeMismatchError("x_a and x_b shapes disagree")


# ---------------------------------------------------------------------------
# Deterministic generator (matrix.py:192-284), vectorized per block kind
# ---------------------------------------------------------------------------

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def _uniform_stream(seed, start, count):
    """Doubles uniform in [-1, 1) from splitmix64 positions start+1..start+count."""
    z = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    z *= _GOLDEN
    z += np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    z ^= z >> np.uint64(30)
    z *= _MIX1
    z ^= z >> np.uint64(27)
    z *= _MIX2
    z ^= z >> np.uint64(31)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -52) - 1.0


def generate_dd_bta(n: int, b: int, a: int, seed: int, dominance: float = 1.5, *, pinned=False) -> BtaMatrix:
    """Deterministic diagonally dominant BT(A) matrix, bit-identical to the
    reference generator (stream order diag, lower, upper, arrow_row,
    arrow_col, tip; each diagonal entry pushed along its phase by
    dominance * (off-diagonal |row| sum + 1)).  For large configurations use
    the device generator (paper_2601_04904_b200.device.generate_dd_bta_device).
    """
    if n < 1 or b < 1 or a < 0:
        raise ValueError(f"invalid shape parameters (n={n}, b={b}, a={a})")
    if dominance < 1.0:
        raise ValueError(f"dominance must be >= 1, got {dominance}")
    m = BtaMatrix.zeros(n, b, a, pinned=pinned)
    pos = 0
    for arr in (m._diag, m._lower, m._upper, m._arrow_row, m._arrow_col, m._tip):
        cnt = arr.size * 2
        if cnt:
            # chunked to bound the uint64 temporaries at large sizes
            flat = arr.reshape(-1)
            step = 1 << 24
            for s in range(0, flat.size, step):
                e = min(flat.size, s + step)
                u = _uniform_stream(seed, pos + 2 * s, 2 * (e - s))
                flat[s:e].real = u[0::2]
                flat[s:e].imag = u[1::2]
        pos += cnt
    _dominance_shift(m, dominance)
    return m


def _dominance_shift(m: BtaMatrix, dominance: float) -> None:
    n, b, a = m.shape_params
    idx = np.arange(b)
    for i in range(n):
        blk = m._diag[i]
        s = np.abs(blk).sum(axis=1) - np.abs(blk[idx, idx])
        if i > 0:
            s += np.abs(m._lower[i - 1]).sum(axis=1)
        if i < n - 1:
            s += np.abs(m._upper[i]).sum(axis=1)
        if a:
            s += np.abs(m._arrow_col[i]).sum(axis=1)
        _push(blk, s, dominance)
    if a:
        s = np.abs(m._tip).sum(axis=1) - np.abs(np.diagonal(m._tip))
        for i in range(n):
            s += np.abs(m._arrow_row[i]).sum(axis=1)
        _push(m._tip, s, dominance)


def _push(block, offsum, dominance):
    k = np.arange(block.shape[0])
    d = block[k, k]
    mag = np.abs(d)
    phase = np.where(mag > 0, d / np.where(mag > 0, mag, 1.0), 1.0)
    block[k, k] = d + dominance * (offsum + 1.0) * phase


def hermitianize(m: BtaMatrix) -> BtaMatrix:
    """``(m + m^H) / 2`` on the pattern (matrix.py:337-354)."""
    out = m.copy()
    H = lambda x: np.conj(np.swapaxes(x, -1, -2))  # noqa: E731
    out._diag[...] = (m._diag + H(m._diag)) / 2.0
    out._upper[...] = (m._upper + H(m._lower)) / 2.0
    out._lower[...] = (m._lower + H(m._upper)) / 2.0
    out._arrow_row[...] = (m._arrow_row + H(m._arrow_col)) / 2.0
    out._arrow_col[...] = (m._arrow_col + H(m._arrow_row)) / 2.0
    out._tip[...] = (m._tip + H(m._tip)) / 2.0
    return out


def to_dense(m) -> np.ndarray:
    """Dense ``N x N`` expansion, zeros off the pattern (matrix.py:292-306)."""
    n, b, a = m.shape_params
    big = np.zeros((n * b + a, n * b + a), dtype=COMPLEX)
    for i in range(n):
        big[i * b:(i + 1) * b, i * b:(i + 1) * b] = m.diag[i]
        big[n * b:, i * b:(i + 1) * b] = m.arrow_row[i]
        big[i * b:(i + 1) * b, n * b:] = m.arrow_col[i]
    for i in range(n - 1):
        big[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b] = m.lower[i]
        big[i * b:(i + 1) * b, (i + 1) * b:(i + 2) * b] = m.upper[i]
    big[n * b:, n * b:] = m.tip
    return big


def mask_to_pattern(dense, shape) -> BtaMatrix:
    """In-pattern entries of a dense array (matrix.py:309-334)."""
    n, b, a = shape
    dense = np.asarray(dense, dtype=COMPLEX)
    if dense.shape != (n * b + a, n * b + a):
        raise ShapeMismatchError(f"dense array has shape {dense.shape}, expected {(n * b + a,) * 2}")
    m = BtaMatrix.zeros(n, b, a)
    for i in range(n):
        m._diag[i] = dense[i * b:(i + 1) * b, i * b:(i + 1) * b]
        m._arrow_row[i] = dense[n * b:, i * b:(i + 1) * b]
        m._arrow_col[i] = dense[i * b:(i + 1) * b, n * b:]
    for i in range(n - 1):
        m._lower[i] = dense[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b]
        m._upper[i] = dense[i * b:(i + 1) * b, (i + 1) * b:(i + 2) * b]
    m._tip[...] = dense[n * b:, n * b:]
    return m
