"""Symmetric backward path (steps.cuh BackSweep): when B = s B^H exactly
(s = +1 Hermitian -- the bench protocol's hermitianize(B), cli.py:273-277;
s = -1 anti-Hermitian -- lesser/greater self-energies), X_B = s X_B^H and the
backward skips the f_l products and the zcol blocks.  The detection is exact
and global (every partition's check is OR-ed); results must match the
reference path (the oracle) to 1e-10 in every case, and the path taken is
visible through Context.b_symmetry()."""

import numpy as np
import pytest
from conftest import max_block_rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200 import _native  # noqa: E402

TOL = 1e-10


def scaled(m, z):
    """Copy of BtaMatrix m times the complex scalar z (exact for z = 1j)."""
    arr = {k: v * z for k, v in m.stacked().items()}
    return bs.BtaMatrix.from_stacked(*m.shape_params, arr, copy=True)


def rhs(n, b, a, kind, seed):
    h = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=seed))
    if kind == "hermitian":
        return h
    if kind == "skew":
        return scaled(h, 1j)
    if kind == "almost":  # Hermitian except one entry of one diagonal block
        arr = {k: v.copy() for k, v in h.stacked().items()}
        arr["diag"][n // 2][1, 0] *= 1.0 + 2.0 ** -40
        return bs.BtaMatrix.from_stacked(n, b, a, arr, copy=False)
    return bs.generate_dd_bta(n, b, a, seed=seed)


EXPECT = {"hermitian": (2, 1), "skew": (1, -1), "almost": (3, 0), "general": (3, 0)}


@pytest.mark.parametrize("kind", ["hermitian", "skew", "almost", "general"])
@pytest.mark.parametrize("n,b,a", [(9, 40, 12), (7, 33, 0), (5, 64, 100)])
def test_sequential_paths(kind, n, b, a):
    A = bs.generate_dd_bta(n, b, a, seed=3)
    B = rhs(n, b, a, kind, seed=4)
    sol = bs.solve_selected(A, B, "siq", partitions=1)
    flags, mode = _native.Context.get(torch.cuda.current_device()).b_symmetry()
    assert (flags, mode) == EXPECT[kind]
    xa, xb = oracle.solve_selected(A, B, "siq")
    assert max_block_rel_err(sol.x_a, xa) <= TOL
    assert max_block_rel_err(sol.x_b, xb) <= TOL
    if kind in ("hermitian", "skew"):
        s = 1 if kind == "hermitian" else -1
        for i in range(n - 1):  # X_B(i+1, i) = s X_B(i, i+1)^H holds exactly on this path
            np.testing.assert_array_equal(sol.x_b.lower[i], s * sol.x_b.upper[i].conj().T)


@pytest.mark.parametrize("kind", ["hermitian", "skew", "general"])
@pytest.mark.parametrize("parts", [2, 3, 5])
def test_partitioned_paths(kind, parts):
    n, b, a = 24, 48, 16
    A = bs.generate_dd_bta(n, b, a, seed=5)
    B = rhs(n, b, a, kind, seed=6)
    got = bs.dist_solve(A, B, num_parts=parts, mode="siq")
    xa, xb = oracle.dist_solve(A, B, num_parts=parts, mode="siq")
    assert max_block_rel_err(got.x_a, xa) <= TOL
    assert max_block_rel_err(got.x_b, xb) <= TOL


def test_one_partition_breaks_symmetry():
    """Only the LAST partition holds the asymmetric entry: every partition
    must take the general path (the decision is global)."""
    n, b, a = 20, 32, 8
    A = bs.generate_dd_bta(n, b, a, seed=7)
    h = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=8))
    arr = {k: v.copy() for k, v in h.stacked().items()}
    arr["lower"][n - 2][0, 3] += 0.25
    B = bs.BtaMatrix.from_stacked(n, b, a, arr)
    got = bs.dist_solve(A, B, num_parts=4, mode="siq")
    xa, xb = oracle.dist_solve(A, B, num_parts=4, mode="siq")
    assert max_block_rel_err(got.x_a, xa) <= TOL
    assert max_block_rel_err(got.x_b, xb) <= TOL


@pytest.mark.parametrize("kind", ["hermitian", "skew", "general"])
def test_streamed_host_inputs(kind):
    """Pinned host inputs streamed in chunks: the chunks are checked as they land."""
    n, b, a = 40, 32, 8
    A = bs.generate_dd_bta(n, b, a, seed=9).copy(pinned=True)
    B = rhs(n, b, a, kind, seed=10).copy(pinned=True)
    sol = bs.solve_selected(A, B, "siq", partitions=2)
    xa, xb = oracle.solve_selected(A, B, "siq")
    assert max_block_rel_err(sol.x_a, xa) <= TOL
    assert max_block_rel_err(sol.x_b, xb) <= TOL


def test_forced_mode_roundtrip():
    ctx = _native.Context.get(torch.cuda.current_device())
    for m in (1, -1, 0, ctx.SYM_AUTO):
        ctx.set_b_symmetry(m)
    with pytest.raises(ValueError):
        ctx.set_b_symmetry(5)


@pytest.fixture
def fused_schur(monkeypatch):
    monkeypatch.setenv("BSEL_SCHUR", "1")  # read by the library per step


@pytest.mark.parametrize("kind", ["hermitian", "general"])
@pytest.mark.parametrize("n,b,a,parts", [(9, 40, 12, 1), (12, 64, 16, 2), (16, 33, 8, 3), (6, 100, 0, 1)])
def test_fused_schur_step_paths(fused_schur, kind, n, b, a, parts):
    A = bs.generate_dd_bta(n, b, a, seed=13)
    B = rhs(n, b, a, kind, seed=14)
    got = bs.dist_solve(A, B, num_parts=parts, mode="siq") if parts > 1 else bs.solve_selected(A, B, "siq",
                                                                                             partitions=1)
    xa, xb = oracle.solve_selected(A, B, "siq")
    assert max_block_rel_err(got.x_a, xa) <= TOL
    assert max_block_rel_err(got.x_b, xb) <= TOL
    got = bs.solve_selected(A, None, "si", partitions=1)
    xa, _ = oracle.solve_selected(A, None, "si")
    assert max_block_rel_err(got.x_a, xa) <= TOL


@pytest.mark.parametrize("b", [40, 64, 96])
@pytest.mark.parametrize("schur", [False, True])
def test_zero_leaf_pivot_fallback(monkeypatch, b, schur):
    """A leaf meeting an exactly zero pivot takes the exact fallback (the
    reference's semantics); with the fused Schur step (inverse + L S +
    C - L S U in one launch) the fallback recomputes S, F, H and the Schur
    complement from the untouched inputs."""
    if schur:
        monkeypatch.setenv("BSEL_SCHUR", "1")
    n, a = 5, 8
    A = bs.generate_dd_bta(n, b, a, seed=11)
    arr = {k: v.copy() for k, v in A.stacked().items()}
    d = arr["diag"][0]
    # first 32 rows of column 0 exactly zero, the block stays nonsingular
    d[:32, 0] = 0.0
    d[b - 1, 0] = 5.0 * b
    A2 = bs.BtaMatrix.from_stacked(n, b, a, arr)
    B = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=12))
    sol = bs.solve_selected(A2, B, "siq", partitions=1)
    xa, xb = oracle.solve_selected(A2, B, "siq")
    assert max_block_rel_err(sol.x_a, xa) <= TOL
    assert max_block_rel_err(sol.x_b, xb) <= TOL


@pytest.mark.parametrize("avoid", [32, 147])
@pytest.mark.parametrize("kind", ["hermitian", "general"])
def test_aux_levels_avoiding_sms(avoid, kind):
    """Forward aux GEMM levels that keep SMs [0, avoid) free (one partition
    per GPU) fetch tiles dynamically; with nearly every SM avoided the last
    CTA to leave works off the tiles -- results unchanged."""
    n, b, a = 9, 72, 20
    A = bs.generate_dd_bta(n, b, a, seed=15)
    B = rhs(n, b, a, kind, seed=16)
    ctx = _native.Context.get(torch.cuda.current_device())
    ctx.set_aux_avoid_sms(avoid)
    try:
        sol = bs.solve_selected(A, B, "siq", partitions=1)
    finally:
        ctx.set_aux_avoid_sms(0)
    xa, xb = oracle.solve_selected(A, B, "siq")
    assert max_block_rel_err(sol.x_a, xa) <= TOL
    assert max_block_rel_err(sol.x_b, xb) <= TOL
