"""Shared fixtures and helpers.

Markers: ``gpu`` tests need a B200 and the built CUDA library; everything
else runs on CPU (oracle vs golden vectors, host logic, C-ABI exports).
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
KINDS = ("diag", "lower", "upper", "arrow_row", "arrow_col")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built libbtasel_b200.so")


def manifest():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


class Stacked:
    """Blocks view over stacked golden arrays (duck-types BtaMatrix)."""

    def __init__(self, z, prefix, n, b, a):
        self.n, self.b, self.a = n, b, a
        for kind in KINDS:
            setattr(self, kind, list(z[f"{prefix}_{kind}"]))
        self.tip = z[f"{prefix}_tip"]

    def blocks(self):
        for kind in KINDS:
            for i, blk in enumerate(getattr(self, kind)):
                yield kind, i, blk
        yield "tip", 0, self.tip


def load_case(name):
    meta = manifest()["cases"][name]
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    n, b, a = meta["n"], meta["b"], meta["a"]
    A = Stacked(z, "a", n, b, a)
    B = Stacked(z, "b", n, b, a) if meta["mode"] == "siq" else None
    XA = Stacked(z, "xa", n, b, a)
    XB = Stacked(z, "xb", n, b, a) if meta["mode"] == "siq" else None
    return meta, A, B, XA, XB


def iter_blocks(m):
    for kind in KINDS:
        for i, blk in enumerate(getattr(m, kind)):
            yield kind, i, np.asarray(blk)
    yield "tip", 0, np.asarray(m.tip)


def max_block_rel_err(cand, ref):
    """Worst per-block relative Frobenius error (reference tests/conftest.py:24-34)."""
    worst = 0.0
    for (_, _, c), (_, _, r) in zip(iter_blocks(cand), iter_blocks(ref)):
        if r.size == 0:
            continue
        den = np.linalg.norm(r)
        err = np.linalg.norm(np.asarray(c) - r)
        worst = max(worst, err / den if den > 0 else err)
    return worst


def identity_block_row_residual(a, x):
    """Dense-free A.X = I check on pattern blocks (reference tests/conftest.py:37-62)."""
    worst = 0.0
    n = a.n
    for j in range(n):
        acc = a.diag[j] @ x.diag[j]
        if j > 0:
            acc = acc + a.lower[j - 1] @ x.upper[j - 1]
        if j < n - 1:
            acc = acc + a.upper[j] @ x.lower[j]
        if a.a:
            acc = acc + a.arrow_col[j] @ x.arrow_row[j]
        worst = max(worst, np.linalg.norm(acc - np.eye(a.b)) / np.sqrt(a.b))
    if a.a:
        acc = a.tip @ x.tip
        for i in range(n):
            acc = acc + a.arrow_row[i] @ x.arrow_col[i]
        worst = max(worst, np.linalg.norm(acc - np.eye(a.a)) / np.sqrt(a.a))
    return worst


def quadratic_block_residual(a, b, xa, xb):
    """Builder-derived dense-free X_B check: the block diagonal of
    A.X_B - B.X_A^H vanishes (pattern blocks only)."""
    H = lambda m: np.conj(m).T  # noqa: E731
    worst = 0.0
    n = a.n
    for j in range(n):
        lhs = a.diag[j] @ xb.diag[j]
        rhs = b.diag[j] @ H(xa.diag[j])
        if j > 0:
            lhs = lhs + a.lower[j - 1] @ xb.upper[j - 1]
            rhs = rhs + b.lower[j - 1] @ H(xa.lower[j - 1])
        if j < n - 1:
            lhs = lhs + a.upper[j] @ xb.lower[j]
            rhs = rhs + b.upper[j] @ H(xa.upper[j])
        if a.a:
            lhs = lhs + a.arrow_col[j] @ xb.arrow_row[j]
            rhs = rhs + b.arrow_col[j] @ H(xa.arrow_col[j])
        worst = max(worst, np.linalg.norm(lhs - rhs) / max(np.linalg.norm(rhs), 1e-300))
    return worst
