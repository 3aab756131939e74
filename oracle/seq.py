"""Sequential oracle: generator, dense bridges and the RGF SI / SI+SQ sweeps.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/btasel/{matrix,kernels,rgf}.py with the same block
products in the same order (so per-step op counts match the reference's
OpCounter exactly), but on a plain `Blocks` record instead of the reference
containers.
"""

from __future__ import annotations

from collections import Counter
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

C128 = np.complex128


class OracleSingular(ArithmeticError):
    """Exact zero pivot; ``index`` is the global diagonal block (n = tip)."""

    def __init__(self, index):
        super().__init__(f"singular pivot at block {index}")
        self.index = index


@dataclass
class Blocks:
    """Pattern blocks of a BT(A) matrix (matrix.py:35-72 layout)."""

    n: int
    b: int
    a: int
    diag: list
    lower: list
    upper: list
    arrow_row: list
    arrow_col: list
    tip: np.ndarray

    @classmethod
    def of(cls, m) -> "Blocks":
        """Deep copy of any object exposing the BtaMatrix attributes."""
        cp = lambda xs: [np.array(x, dtype=C128, copy=True) for x in xs]  # noqa: E731
        return cls(m.n, m.b, m.a, cp(m.diag), cp(m.lower), cp(m.upper), cp(m.arrow_row),
                   cp(m.arrow_col), np.array(m.tip, dtype=C128, copy=True))

    @classmethod
    def zeros(cls, n, b, a) -> "Blocks":
        z = lambda k, r, c: [np.zeros((r, c), C128) for _ in range(k)]  # noqa: E731
        return cls(n, b, a, z(n, b, b), z(n - 1, b, b), z(n - 1, b, b), z(n, a, b), z(n, b, a),
                   np.zeros((a, a), C128))

    def blocks(self):
        """(kind, index, block) in the reference's pattern order (matrix.py:141-153)."""
        for kind in ("diag", "lower", "upper", "arrow_row", "arrow_col"):
            for i, blk in enumerate(getattr(self, kind)):
                yield kind, i, blk
        yield "tip", 0, self.tip


# ---------------------------------------------------------------------------
# Counting product helper (kernels.py:37-166)
# ---------------------------------------------------------------------------


class _Mul:
    """op(x) @ op(y) with shape-class tallies (kernels.py:55-71)."""

    def __init__(self, b, a):
        self.b, self.a = b, a
        self.counts = Counter()
        self.inverses = 0

    def _cls(self, d):
        return "b" if d == self.b else ("a" if d == self.a else "?")

    def __call__(self, x, y, hx=False, hy=False):
        x = x.conj().T if hx else x
        y = y.conj().T if hy else y
        m, k = x.shape
        n = y.shape[1]
        if m and k and n:
            self.counts[self._cls(m) + self._cls(k) + self._cls(n)] += 1
        return x @ y

    def inv(self, blk, index):
        """LU with partial pivoting + solve against I (kernels.py:169-236,
        rgf.py:64-71); exact zero U pivot -> OracleSingular(index)."""
        self.inverses += 1
        if blk.shape[0] == 0:
            return np.zeros((0, 0), C128)
        lu, piv = scipy.linalg.lu_factor(blk, check_finite=False)
        if np.any(np.diagonal(lu) == 0):
            raise OracleSingular(index)
        return scipy.linalg.lu_solve((lu, piv), np.eye(blk.shape[0], dtype=C128), check_finite=False)


# ---------------------------------------------------------------------------
# Deterministic generator (matrix.py:192-284)
# ---------------------------------------------------------------------------

_M64 = (1 << 64) - 1


def _splitmix_block(seed, offset, rows, cols):
    """Complex block from the splitmix64 stream positions offset+1 .. offset+2rc
    (matrix.py:197-221): re/im interleaved, uniform in [-1, 1)."""
    cnt = 2 * rows * cols
    if cnt == 0:
        return np.zeros((rows, cols), C128)
    pos = np.arange(offset + 1, offset + cnt + 1, dtype=np.uint64)
    z = np.uint64(seed & _M64) + pos * np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    u = 2.0 * ((z >> np.uint64(11)).astype(np.float64) * 2.0**-53) - 1.0
    return (u[0::2] + 1j * u[1::2]).reshape(rows, cols)


def _boost(block, offsum, dominance):
    """Shift each diagonal entry along its phase (matrix.py:262-267)."""
    k = np.arange(block.shape[0])
    d = block[k, k]
    mag = np.abs(d)
    unit = np.where(mag > 0, d / np.where(mag > 0, mag, 1.0), 1.0)
    block[k, k] = d + dominance * (offsum + 1.0) * unit


def generate_dd_bta(n, b, a, seed, dominance=1.5) -> Blocks:
    """matrix.py:224-284: stream order diag, lower, upper, arrow_row,
    arrow_col, tip; then row-dominance shift of every diagonal entry."""
    off = 0
    out = []
    for count, r, c in ((n, b, b), (n - 1, b, b), (n - 1, b, b), (n, a, b), (n, b, a), (1, a, a)):
        lst = []
        for _ in range(count):
            lst.append(_splitmix_block(seed, off, r, c))
            off += 2 * r * c
        out.append(lst)
    m = Blocks(n, b, a, out[0], out[1], out[2], out[3], out[4], out[5][0])
    for i in range(n):
        s = np.abs(m.diag[i]).sum(axis=1) - np.abs(np.diagonal(m.diag[i]))
        if i > 0:
            s += np.abs(m.lower[i - 1]).sum(axis=1)
        if i < n - 1:
            s += np.abs(m.upper[i]).sum(axis=1)
        if a:
            s += np.abs(m.arrow_col[i]).sum(axis=1)
        _boost(m.diag[i], s, dominance)
    if a:
        s = np.abs(m.tip).sum(axis=1) - np.abs(np.diagonal(m.tip))
        for i in range(n):
            s += np.abs(m.arrow_row[i]).sum(axis=1)
        _boost(m.tip, s, dominance)
    return m


def hermitianize(m) -> Blocks:
    """(m + m^H)/2 on the pattern (matrix.py:337-354)."""
    x = Blocks.of(m)
    h = lambda p, q: (p + q.conj().T) / 2.0  # noqa: E731
    x.diag = [h(d, d) for d in m.diag]
    x.upper = [h(u, lo) for u, lo in zip(m.upper, m.lower)]
    x.lower = [h(lo, u) for u, lo in zip(m.upper, m.lower)]
    x.arrow_row = [h(r, c) for r, c in zip(m.arrow_row, m.arrow_col)]
    x.arrow_col = [h(c, r) for r, c in zip(m.arrow_row, m.arrow_col)]
    x.tip = h(m.tip, m.tip)
    return x


def to_dense(m) -> np.ndarray:
    """matrix.py:292-306."""
    n, b, a = m.n, m.b, m.a
    out = np.zeros((n * b + a, n * b + a), C128)
    sl = lambda i: slice(i * b, (i + 1) * b)  # noqa: E731
    for i in range(n):
        out[sl(i), sl(i)] = m.diag[i]
        out[n * b:, sl(i)] = m.arrow_row[i]
        out[sl(i), n * b:] = m.arrow_col[i]
    for i in range(n - 1):
        out[sl(i + 1), sl(i)] = m.lower[i]
        out[sl(i), sl(i + 1)] = m.upper[i]
    out[n * b:, n * b:] = m.tip
    return out


def mask_to_pattern(dense, n, b, a) -> Blocks:
    """matrix.py:309-334."""
    sl = lambda i: slice(i * b, (i + 1) * b)  # noqa: E731
    t = slice(n * b, n * b + a)
    return Blocks(
        n, b, a,
        [dense[sl(i), sl(i)].copy() for i in range(n)],
        [dense[sl(i + 1), sl(i)].copy() for i in range(n - 1)],
        [dense[sl(i), sl(i + 1)].copy() for i in range(n - 1)],
        [dense[t, sl(i)].copy() for i in range(n)],
        [dense[sl(i), t].copy() for i in range(n)],
        dense[t, t].copy(),
    )


def dense_selected(a, b=None):
    """Independent dense oracle (tests/conftest.py:13-21): inv(A) and
    inv(A) B inv(A)^H masked to the pattern."""
    inv = np.linalg.inv(to_dense(a))
    xa = mask_to_pattern(inv, a.n, a.b, a.a)
    xb = None if b is None else mask_to_pattern(inv @ to_dense(b) @ inv.conj().T, a.n, a.b, a.a)
    return xa, xb


# ---------------------------------------------------------------------------
# Forward sweeps (rgf.py:79-124, 207-319)
# ---------------------------------------------------------------------------


@dataclass
class Factors:
    """rgf.py:37-61."""

    n: int
    b: int
    a: int
    fused: bool
    s_a: list = field(default_factory=list)
    s_b: list = field(default_factory=list)
    b_diag_last: np.ndarray | None = None
    ar_e: list = field(default_factory=list)
    ac_e: list = field(default_factory=list)
    br_e: list = field(default_factory=list)
    bc_e: list = field(default_factory=list)
    tip_inv: np.ndarray | None = None
    b_tip: np.ndarray | None = None


def forward(A: Blocks, B: Blocks | None, mul: _Mul) -> Factors:
    """In-place forward Schur sweep on working copies A (and B)."""
    n, a = A.n, A.a
    fz = B is not None
    F = Factors(n, A.b, a, fz)
    F.s_a = [None] * n
    F.s_b = [None] * max(n - 1, 0)
    if a == 0:
        # rgf.py:104-123
        for i in range(n - 1):
            S = mul.inv(A.diag[i], i)
            F.s_a[i] = S
            t1 = mul(A.lower[i], S)
            if fz:
                sb = mul(mul(S, B.diag[i]), S, hy=True)
                F.s_b[i] = sb
                v = mul(A.lower[i], sb)
                B.diag[i + 1] = (B.diag[i + 1] + mul(v, A.lower[i], hy=True)
                                 - mul(B.lower[i], t1, hy=True) - mul(t1, B.upper[i]))
            A.diag[i + 1] = A.diag[i + 1] - mul(t1, A.upper[i])
        F.s_a[n - 1] = mul.inv(A.diag[n - 1], n - 1)
        if fz:
            F.b_diag_last = B.diag[n - 1].copy()
        return F

    F.ar_e, F.ac_e = [None] * n, [None] * n
    F.br_e, F.bc_e = [None] * n, [None] * n
    for i in range(n):
        S = mul.inv(A.diag[i], i)
        F.s_a[i] = S
        F.ar_e[i], F.ac_e[i] = A.arrow_row[i], A.arrow_col[i]
        if fz:
            F.br_e[i], F.bc_e[i] = B.arrow_row[i], B.arrow_col[i]
        last = i == n - 1
        if not fz:
            if last:  # rgf.py:311-312
                t2 = mul(S, A.arrow_col[i])
                A.tip = A.tip - mul(A.arrow_row[i], t2)
                break
            # rgf.py:283-288
            t1 = mul(S, A.upper[i])
            t2 = mul(S, A.arrow_col[i])
            A.diag[i + 1] = A.diag[i + 1] - mul(A.lower[i], t1)
            A.arrow_row[i + 1] = A.arrow_row[i + 1] - mul(A.arrow_row[i], t1)
            A.arrow_col[i + 1] = A.arrow_col[i + 1] - mul(A.lower[i], t2)
            A.tip = A.tip - mul(A.arrow_row[i], t2)
            continue
        if last:  # rgf.py:297-309
            F.b_diag_last = B.diag[i].copy()
            g = mul(A.arrow_row[i], S)
            p = mul(g, B.diag[i])
            A.tip = A.tip - mul(g, A.arrow_col[i])
            B.tip = (B.tip - mul(g, B.arrow_col[i]) - mul(B.arrow_row[i], g, hy=True)
                     + mul(p, g, hy=True))
            F.b_tip = B.tip.copy()
            break
        # rgf.py:246-280
        Bd = B.diag[i]
        sb = mul(mul(S, Bd), S, hy=True)
        F.s_b[i] = sb
        f = mul(A.lower[i], S)
        g = mul(A.arrow_row[i], S)
        p = mul(g, Bd)
        k = mul(Bd, g, hy=True)
        A.diag[i + 1] = A.diag[i + 1] - mul(f, A.upper[i])
        A.arrow_row[i + 1] = A.arrow_row[i + 1] - mul(g, A.upper[i])
        A.arrow_col[i + 1] = A.arrow_col[i + 1] - mul(f, A.arrow_col[i])
        A.tip = A.tip - mul(g, A.arrow_col[i])
        v = mul(A.lower[i], sb)
        B.diag[i + 1] = (B.diag[i + 1] + mul(v, A.lower[i], hy=True) - mul(B.lower[i], f, hy=True)
                         - mul(f, B.upper[i]))
        B.arrow_row[i + 1] = (B.arrow_row[i + 1] - mul(g, B.upper[i])
                              + mul(p - B.arrow_row[i], f, hy=True))
        B.arrow_col[i + 1] = (B.arrow_col[i + 1] - mul(f, B.arrow_col[i])
                              - mul(B.lower[i], g, hy=True) + mul(f, k))
        B.tip = (B.tip - mul(g, B.arrow_col[i]) - mul(B.arrow_row[i], g, hy=True)
                 + mul(p, g, hy=True))
    F.tip_inv = mul.inv(A.tip, n)  # rgf.py:313-318
    return F


# ---------------------------------------------------------------------------
# Backward sweeps (rgf.py:127-199, 322-489)
# ---------------------------------------------------------------------------


def backstep(mul, g, rs, qs, ya, sc=None, ss=None, ws=None, yb=None):
    """Generic Takahashi step with k trailing couplings (rgf.py:322-398).

    Returns (row, col, diag) for X_A and, when the quadratic data is given,
    (row, col, diag) for X_B.  Products are issued in the reference order.
    """
    k = len(rs)
    ks = range(k)

    def chain(pairs):
        acc = None
        for x, y, hx, hy in pairs:
            t = mul(x, y, hx, hy)
            acc = t if acc is None else acc + t
        return acc

    row = [-mul(g, chain((rs[l], ya[l][j], 0, 0) for l in ks)) for j in ks]
    col = [-mul(chain((ya[j][l], qs[l], 0, 0) for l in ks), g) for j in ks]
    phi = -mul(row[0], qs[0])
    for l in range(1, k):
        phi = phi - mul(row[l], qs[l])
    dia = g + mul(phi, g)
    if yb is None:
        return (row, col, dia), None

    e = [mul(g, ss[l]) - mul(sc, qs[l], hy=True) for l in ks]
    f = [mul(ws[l], g, hy=True) - mul(qs[l], sc) for l in ks]
    zrow = [chain((e[l], ya[j][l], 0, 1) for l in ks) - mul(g, chain((rs[l], yb[l][j], 0, 0) for l in ks))
            for j in ks]
    zcol = [chain((ya[j][l], f[l], 0, 0) for l in ks)
            - mul(chain((yb[j][l], rs[l], 0, 1) for l in ks), g, hy=True) for j in ks]
    zd = sc + mul(phi, sc) + mul(sc, phi, hy=True)
    zd = zd + mul(g, chain((ss[l], row[l], 0, 1) for l in ks))
    zd = zd + mul(chain((row[l], ws[l], 0, 0) for l in ks), g, hy=True)
    quad = None
    for l in ks:
        t = mul(rs[l], chain((yb[l][m], rs[m], 0, 1) for m in ks))
        quad = t if quad is None else quad + t
    zd = zd + mul(mul(g, quad), g, hy=True)
    return (row, col, dia), (zrow, zcol, zd)


def backward(F: Factors, A: Blocks, B: Blocks | None, mul: _Mul, diagonal_only=False):
    """Returns (X_A, X_B) as Blocks; X_B None in SI mode."""
    n, bs, a = F.n, F.b, F.a
    fz = F.fused
    XA = Blocks.zeros(n, bs, a)
    XB = Blocks.zeros(n, bs, a) if fz else None
    if a == 0:
        # rgf.py:156-197
        xd = F.s_a[n - 1].copy()
        XA.diag[n - 1] = xd
        if fz:
            zd = mul(mul(F.s_a[n - 1], F.b_diag_last), F.s_a[n - 1], hy=True)
            XB.diag[n - 1] = zd
        for i in range(n - 2, -1, -1):
            S, xp = F.s_a[i], xd
            tA1 = mul(S, A.upper[i])
            tA2 = mul(xp, A.lower[i])
            xlo = -mul(tA2, S)
            xup = -mul(tA1, xp)
            xd = S - mul(tA1, xlo)
            XA.diag[i] = xd
            if not diagonal_only:
                XA.lower[i], XA.upper[i] = xlo, xup
            if fz:
                zp, sb = zd, F.s_b[i]
                tB1 = mul(zp, tA1, hy=True)
                tB2 = mul(sb, tA2, hy=True)
                tB3 = mul(tA2, sb)
                tB4 = mul(mul(S, B.upper[i]), xp, hy=True)
                tB5 = mul(mul(xp, B.lower[i]), S, hy=True)
                zup = -mul(tA1, zp) - tB2 + tB4
                zlo = -tB1 - tB3 + tB5
                zd = (sb + mul(tA1, tB1) + mul(tA1, tB3) + mul(tB2, tA1, hy=True)
                      - mul(tA1, tB5) - mul(tB4, tA1, hy=True))
                XB.diag[i] = zd
                if not diagonal_only:
                    XB.lower[i], XB.upper[i] = zlo, zup
        return XA, XB

    # rgf.py:428-487
    ytt = F.tip_inv
    XA.tip = ytt.copy()
    ztt = None
    if fz:
        ztt = mul(mul(ytt, F.b_tip), ytt, hy=True)
        XB.tip = ztt.copy()
    prev = None
    for i in range(n - 1, -1, -1):
        if i == n - 1:
            rs, qs, ya = [F.ac_e[i]], [F.ar_e[i]], [[ytt]]
            if fz:
                ss, ws, yb = [F.bc_e[i]], [F.br_e[i]], [[ztt]]
                sc = mul(mul(F.s_a[i], F.b_diag_last), F.s_a[i], hy=True)
        else:
            (ydd, ydt, ytd), zprev = prev
            rs, qs = [A.upper[i], F.ac_e[i]], [A.lower[i], F.ar_e[i]]
            ya = [[ydd, ydt], [ytd, ytt]]
            if fz:
                zdd, zdt, ztd = zprev
                ss, ws = [B.upper[i], F.bc_e[i]], [B.lower[i], F.br_e[i]]
                yb = [[zdd, zdt], [ztd, ztt]]
                sc = F.s_b[i]
        if fz:
            xa, xb = backstep(mul, F.s_a[i], rs, qs, ya, sc, ss, ws, yb)
        else:
            xa, xb = backstep(mul, F.s_a[i], rs, qs, ya)
        row, col, dia = xa
        XA.diag[i], XA.arrow_col[i], XA.arrow_row[i] = dia, row[-1], col[-1]
        if i < n - 1 and not diagonal_only:
            XA.upper[i], XA.lower[i] = row[0], col[0]
        zstate = None
        if fz:
            zr, zc, zdg = xb
            XB.diag[i], XB.arrow_col[i], XB.arrow_row[i] = zdg, zr[-1], zc[-1]
            if i < n - 1 and not diagonal_only:
                XB.upper[i], XB.lower[i] = zr[0], zc[0]
            zstate = (zdg, zr[-1], zc[-1])
        prev = ((dia, row[-1], col[-1]), zstate)
    return XA, XB


def solve_selected(a, b=None, mode=None, *, diagonal_only=False, counts=None):
    """Non-destructive facade (rgf.py:497-531).  Returns (X_A, X_B)."""
    if mode is None:
        mode = "si" if b is None else "siq"
    if mode not in ("si", "siq"):
        raise ValueError(f"mode must be 'si' or 'siq', got {mode!r}")
    if mode == "siq" and b is None:
        raise ValueError("mode 'siq' requires a right-hand side")
    A = Blocks.of(a)
    B = Blocks.of(b) if mode == "siq" else None
    mul = _Mul(A.b, A.a)
    F = forward(A, B, mul)
    out = backward(F, A, B, mul, diagonal_only)
    if counts is not None:
        counts.update(mul.counts)
    return out


def op_counts(n, b, a, mode, forward_only=False):
    """Shape-class product tallies of one sequential solve, measured by
    running the oracle on tiny blocks of the same (n, b, a) classes."""
    bb, aa = (3, 2) if a else (3, 0)
    A = generate_dd_bta(n, bb, aa, seed=1)
    B = hermitianize(generate_dd_bta(n, bb, aa, seed=2)) if mode == "siq" else None
    mul = _Mul(bb, aa)
    F = forward(Blocks.of(A), None if B is None else Blocks.of(B), mul)
    if not forward_only:
        backward(F, A, B, mul)
    return dict(mul.counts), mul.inverses
