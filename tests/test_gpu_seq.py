"""GPU parity of the sequential path (C ABI -> sm_100a kernels) against the
CPU oracle and the reference golden vectors.  Tolerance: 1e-10 max per-block
relative Frobenius error (BASELINE.json north star), complex128."""

import numpy as np
import pytest
from conftest import (identity_block_row_residual, load_case, manifest, max_block_rel_err,
                      quadratic_block_residual)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200 import _native  # noqa: E402

TOL = 1e-10
rng = np.random.default_rng(20240901)


def crand(*shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# --------------------------------------------------------------------------
# kernels: grouped DMMA ZGEMM and block inverse
# --------------------------------------------------------------------------


@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (3, 5, 2), (17, 33, 9), (64, 64, 64), (100, 37, 129),
                                   (256, 512, 64), (512, 512, 512)])
@pytest.mark.parametrize("ta", [False, True])
@pytest.mark.parametrize("tb", [False, True])
def test_zgemm_vs_numpy(m, k, n, ta, tb):
    a = crand(k, m) if ta else crand(m, k)
    b = crand(n, k) if tb else crand(k, n)
    c = crand(m, n)
    opa = a.conj().T if ta else a
    opb = b.conj().T if tb else b
    ref = opa @ opb
    got = bs.block_multiply_acc(None, a, b, trans_a=ta, trans_b=tb)
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref) * max(1, np.sqrt(k))
    got = bs.block_multiply_acc(c, a, b, alpha=-1.0, beta=1.0, trans_a=ta, trans_b=tb)
    ref2 = c - ref
    assert np.linalg.norm(got - ref2) <= 1e-13 * np.linalg.norm(ref2) * max(1, np.sqrt(k))


def test_zgemm_general_alpha_beta_and_counter():
    a, b, c = crand(7, 4), crand(4, 5), crand(7, 5)
    cnt = bs.OpCounter(b=7, a=4)
    got = bs.block_multiply_acc(c, a, b, alpha=0.5 - 2j, beta=1.5j, counter=cnt)
    np.testing.assert_allclose(got, 1.5j * c + (0.5 - 2j) * (a @ b), rtol=1e-13, atol=1e-13)
    assert dict(cnt.gemm_by_shape) == {"ba?": 1}
    with pytest.raises(bs.ShapeMismatchError):
        bs.block_multiply_acc(None, crand(3, 4), crand(5, 2))


@pytest.mark.parametrize("n", [1, 2, 5, 31, 32, 33, 64, 100, 256, 512, 1000, 1024])
def test_block_inverse_dd(n):
    x = crand(n, n) + np.diag(3.0 * n * np.ones(n))
    got = bs.block_inverse(x)
    res = np.linalg.norm(x @ got - np.eye(n)) / np.sqrt(n)
    assert res <= 1e-13
    np.testing.assert_allclose(got, np.linalg.inv(x), rtol=1e-11, atol=1e-14)


def test_block_inverse_repeated_sizes():
    """The dataflow inverse's ready flags are epoch-tagged and never reset:
    back-to-back launches of different sizes on one workspace stay exact."""
    for n in (512, 96, 512, 1000, 64, 512):
        x = crand(n, n) + np.diag(3.0 * n * np.ones(n))
        got = bs.block_inverse(x)
        np.testing.assert_allclose(got, np.linalg.inv(x), rtol=1e-11, atol=1e-14)


@pytest.mark.parametrize("n", [2, 7, 40, 96])
def test_block_inverse_needs_pivoting(n):
    # Non-DD: zero leading leaf pivots -> exact partial-pivoting fallback path.
    x = crand(n, n)
    x[:, 0] *= 0.0
    x[n - 1, 0] = 1.0 + 0.5j
    x[0, :] = 0.0
    x[0, n - 1] = 2.0
    got = bs.block_inverse(x)
    assert np.linalg.norm(x @ got - np.eye(n)) / np.sqrt(n) <= 1e-10


@pytest.mark.parametrize("n", [64, 96, 512])
def test_block_inverse_small_in_tile_pivot(n):
    """A nonsingular block whose leading 32-row tile has only tiny entries in
    its first columns while rows below hold O(1) ones: pivoting inside the
    diagonal tile alone would pick a ~1e-12 pivot (growth 1e12); the growth
    check (block multipliers > 16) hands the block to the exact full-column
    partial-pivoting inverse -> LAPACK accuracy."""
    x = crand(n, n)
    x[:32, :4] *= 1e-12
    got = bs.block_inverse(x)
    ref = np.linalg.inv(x)
    assert np.linalg.norm(got - ref) <= 1e-9 * np.linalg.norm(ref)
    assert np.linalg.norm(x @ got - np.eye(n)) / np.sqrt(n) <= 1e-9


def test_block_inverse_singular_reports_row():
    x = np.eye(4, dtype=np.complex128)
    x[2, :] = 0.0
    x[:, 2] = 0.0
    with pytest.raises(bs.SingularBlockError) as info:
        bs.block_inverse(x)
    assert info.value.index == 2
    np.testing.assert_allclose(bs.block_inverse(np.array([[2.0, 1.0], [1.0, 2.0]])),
                               [[2 / 3, -1 / 3], [-1 / 3, 2 / 3]], rtol=1e-14)


@pytest.mark.parametrize("n,r", [(96, 50), (512, 300)])
def test_block_inverse_singular_dataflow(n, r):
    """Multi-panel blocks go through the dataflow kernel, whose exact fallback
    runs inside the kernel: an exactly singular block is still reported with
    its pivot row, and the next inverse on the same workspace is exact."""
    x = crand(n, n) + np.diag(3.0 * n * np.ones(n))
    x[r, :] = 0.0
    x[:, r] = 0.0
    with pytest.raises(bs.SingularBlockError) as info:
        bs.block_inverse(x)
    assert info.value.index == r
    y = crand(n, n) + np.diag(3.0 * n * np.ones(n))
    np.testing.assert_allclose(bs.block_inverse(y), np.linalg.inv(y), rtol=1e-11, atol=1e-14)


@pytest.mark.parametrize("grid", [2, 3, 7, 40, 148])
def test_block_inverse_grid_sizes(grid):
    """Dataflow inverse with 1 .. 147 worker CTAs (tile ranges of 256 .. 2
    tiles, ragged last ranges, empty ranges) and a ragged block size."""
    ctx = _native.Context.get()
    ctx.set_inverse_grid(grid)
    try:
        for n in (512, 200):
            x = crand(n, n) + np.diag(3.0 * n * np.ones(n))
            np.testing.assert_allclose(bs.block_inverse(x), np.linalg.inv(x), rtol=1e-11, atol=1e-14)
    finally:
        ctx.set_inverse_grid(0)


# --------------------------------------------------------------------------
# solver vs reference golden vectors and oracle
# --------------------------------------------------------------------------

M = manifest()
SEQ = sorted(k for k, v in M["cases"].items() if v["kind"] == "seq")


@pytest.mark.parametrize("name", SEQ)
def test_solve_selected_vs_reference_golden(name):
    meta, A, B, XA, XB = load_case(name)
    a = bs.BtaMatrix(A.n, A.b, A.a, A.diag, A.lower, A.upper, A.arrow_row, A.arrow_col, A.tip)
    b = None
    if B is not None:
        b = bs.BtaMatrix(B.n, B.b, B.a, B.diag, B.lower, B.upper, B.arrow_row, B.arrow_col, B.tip)
    cnt = bs.OpCounter(b=A.b, a=A.a)
    sol = bs.solve_selected(a, b, meta["mode"], counter=cnt)
    assert max_block_rel_err(sol.x_a, XA) <= TOL
    if XB is not None:
        assert max_block_rel_err(sol.x_b, XB) <= TOL
    assert cnt.as_dict() == meta["counts"]


GRID = [(n, b, a) for n in (1, 2, 3, 7) for b in (1, 3) for a in (0, 1, 4)]


@pytest.mark.parametrize("n,b,a", GRID)
def test_property_grid_vs_dense(n, b, a):
    A = bs.generate_dd_bta(n, b, a, seed=n * 100 + b * 10 + a)
    B = bs.generate_dd_bta(n, b, a, seed=n * 100 + b * 10 + a + 1_000_003)
    sol = bs.solve_selected(A, B, "siq")
    da, db = oracle.dense_selected(A, B)
    assert max_block_rel_err(sol.x_a, da) <= TOL
    assert max_block_rel_err(sol.x_b, db) <= TOL


SHAPES = [
    (4, 64, 0, "si"), (4, 64, 0, "siq"), (5, 96, 40, "si"), (5, 96, 40, "siq"),
    (3, 100, 33, "siq"), (6, 128, 16, "siq"), (3, 40, 100, "siq"), (4, 64, 64, "siq"),
]


@pytest.mark.parametrize("n,b,a,mode", SHAPES)
def test_solve_selected_vs_oracle(n, b, a, mode):
    A = bs.generate_dd_bta(n, b, a, seed=7)
    B = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=8)) if mode == "siq" else None
    sol = bs.solve_selected(A, B, mode)
    xa, xb = oracle.solve_selected(A, B, mode)
    assert max_block_rel_err(sol.x_a, xa) <= TOL
    if mode == "siq":
        assert max_block_rel_err(sol.x_b, xb) <= TOL


def test_config1_bt_si_n16_b64():
    """BASELINE config 1, bench protocol inputs, vs oracle and the reference digest."""
    A = bs.generate_dd_bta(16, 64, 0, seed=0)
    sol = bs.solve_selected(A)
    xa, _ = oracle.solve_selected(A)
    assert max_block_rel_err(sol.x_a, xa) <= TOL
    norms = [np.linalg.norm(blk) for _, _, blk in sol.x_a.pattern_blocks() if blk.size]
    np.testing.assert_allclose(norms, M["config1_digest"]["norm"], rtol=1e-12)


def test_config2_bt_siq_n64_b256():
    """BASELINE config 2 at full size vs the oracle."""
    A = bs.generate_dd_bta(64, 256, 0, seed=0)
    B = bs.hermitianize(bs.generate_dd_bta(64, 256, 0, seed=1))
    sol = bs.solve_selected(A, B)
    xa, xb = oracle.solve_selected(A, B)
    assert max_block_rel_err(sol.x_a, xa) <= TOL
    assert max_block_rel_err(sol.x_b, xb) <= TOL


def test_config3_shape_bta_siq_b512_a64():
    """BASELINE config 3 shapes (b=512, a=64) at n=12 vs the oracle, plus
    dense-free residuals at the full n=128 on the GPU output."""
    A = bs.generate_dd_bta(12, 512, 64, seed=0)
    B = bs.hermitianize(bs.generate_dd_bta(12, 512, 64, seed=1))
    sol = bs.solve_selected(A, B)
    xa, xb = oracle.solve_selected(A, B)
    assert max_block_rel_err(sol.x_a, xa) <= TOL
    assert max_block_rel_err(sol.x_b, xb) <= TOL


def test_config3_full_dense_free_residuals():
    A = bs.generate_dd_bta(128, 512, 64, seed=0)
    B = bs.hermitianize(bs.generate_dd_bta(128, 512, 64, seed=1))
    dA, dB = bs.to_device(A), bs.to_device(B)
    sol = bs.solve_selected(dA, dB)
    xa, xb = bs.to_host(sol.x_a), bs.to_host(sol.x_b)
    assert identity_block_row_residual(A, xa) <= 1e-12
    assert quadratic_block_residual(A, B, xa, xb) <= 1e-11


def test_forward_backward_split_matches_facade():
    A = bs.generate_dd_bta(5, 24, 8, seed=3)
    B = bs.hermitianize(bs.generate_dd_bta(5, 24, 8, seed=4))
    full = bs.solve_selected(A, B)
    wa, wb = A.copy(), B.copy()
    f = bs.bta_forward(wa, wb)
    assert len(f.s_a) == 5 and f.tip_schur_inv.shape == (8, 8)
    sol = bs.bta_backward(f, wa, wb)
    assert max_block_rel_err(sol.x_a, full.x_a) <= 1e-13
    assert max_block_rel_err(sol.x_b, full.x_b) <= 1e-13
    # backward from host-only factors (re-upload path)
    f._dev = None
    sol2 = bs.bta_backward(f, wa, wb)
    assert max_block_rel_err(sol2.x_b, full.x_b) <= 1e-13


def test_determinism_and_non_mutation():
    A = bs.generate_dd_bta(6, 40, 12, seed=11)
    B = bs.generate_dd_bta(6, 40, 12, seed=12)
    a0, b0 = A.copy(), B.copy()
    s1 = bs.solve_selected(A, B, "siq")
    s2 = bs.solve_selected(A, B, "siq")
    assert s1.x_a.equals_exact(s2.x_a) and s1.x_b.equals_exact(s2.x_b)
    assert A.equals_exact(a0) and B.equals_exact(b0)


def test_a0_bta_path_is_bitwise_bt():
    A = bs.generate_dd_bta(5, 33, 0, seed=5)
    B = bs.generate_dd_bta(5, 33, 0, seed=6)
    wa1, wb1 = A.copy(), B.copy()
    s1 = bs.bta_backward(bs.bta_forward(wa1, wb1), wa1, wb1)
    wa2, wb2 = A.copy(), B.copy()
    s2 = bs.bt_backward(bs.bt_forward(wa2, wb2), wa2, wb2)
    assert s1.x_a.equals_exact(s2.x_a) and s1.x_b.equals_exact(s2.x_b)


def test_identity_and_known_answers():
    a = bs.BtaMatrix.identity(3, 2)
    b = bs.generate_dd_bta(3, 2, 0, seed=2)
    sol = bs.solve_selected(a, b)
    assert sol.x_a.equals_exact(bs.BtaMatrix.identity(3, 2))
    assert max_block_rel_err(sol.x_b, b) == 0.0
    two = bs.BtaMatrix(2, 1, 0, [[[2.0]], [[2.0]]], [[[1.0]]], [[[1.0]]])
    np.testing.assert_allclose(bs.to_dense(bs.solve_selected(two).x_a), [[2 / 3, -1 / 3], [-1 / 3, 2 / 3]],
                               rtol=1e-14)
    f = bs.bt_forward(two.copy())
    np.testing.assert_allclose([s[0, 0] for s in f.s_a], [0.5, 1 / 1.5], rtol=1e-14)
    arrow = bs.BtaMatrix(1, 1, 1, [[[2.0]]], [], [], [[[1.0]]], [[[1.0]]], [[3.0]])
    f = bs.bta_forward(arrow.copy())
    np.testing.assert_allclose(f.tip_schur_inv, [[1 / 2.5]], rtol=1e-14)
    np.testing.assert_allclose(bs.to_dense(bs.solve_selected(arrow).x_a), [[0.6, -0.2], [-0.2, 0.4]],
                               rtol=1e-14)
    ident = bs.BtaMatrix.identity(3, 2, 2)
    assert bs.solve_selected(ident).x_a.equals_exact(bs.BtaMatrix.identity(3, 2, 2))


def test_singular_pivot_and_tip_indices():
    a = bs.BtaMatrix.identity(3, 2)
    a.diag[1][:] = 0.0
    with pytest.raises(bs.SingularBlockError) as info:
        bs.bt_forward(a.copy())
    assert info.value.index == 1
    a = bs.BtaMatrix.identity(2, 2, 1)
    a.tip[:] = 0.0
    with pytest.raises(bs.SingularBlockError) as info:
        bs.solve_selected(a)
    assert info.value.index == 2
    # a non-DD but nonsingular pivot needing row interchanges is fine
    p = bs.BtaMatrix(1, 2, 0, [[[0.0, 1.0], [1.0, 0.0]]], [], [])
    np.testing.assert_allclose(bs.solve_selected(p).x_a.diag[0], [[0, 1], [1, 0]], atol=1e-15)


def test_diagonal_only_and_hermitian_preservation():
    A = bs.generate_dd_bta(6, 20, 6, seed=12)
    B = bs.hermitianize(bs.generate_dd_bta(6, 20, 6, seed=13))
    full = bs.solve_selected(A, B)
    diag = bs.solve_selected(A, B, diagonal_only=True)
    for i in range(6):
        np.testing.assert_array_equal(diag.x_a.diag[i], full.x_a.diag[i])
    assert all(np.all(blk == 0) for blk in diag.x_a.lower)
    assert all(np.all(blk == 0) for blk in diag.x_b.upper)
    x = full.x_b
    scale = max(np.linalg.norm(blk) for _, _, blk in x.pattern_blocks() if blk.size)
    for i in range(x.n):
        assert np.linalg.norm(x.diag[i] - x.diag[i].conj().T) <= 1e-12 * scale
        assert np.linalg.norm(x.arrow_col[i] - x.arrow_row[i].conj().T) <= 1e-12 * scale
    for i in range(x.n - 1):
        assert np.linalg.norm(x.upper[i] - x.lower[i].conj().T) <= 1e-12 * scale


def test_timings_and_device_path():
    A = bs.generate_dd_bta(8, 64, 16, seed=14)
    B = bs.hermitianize(bs.generate_dd_bta(8, 64, 16, seed=15))
    dA, dB = bs.to_device(A), bs.to_device(B)
    t = {}
    sol = bs.solve_selected(dA, dB, timings=t)
    assert set(t) == {"forward", "backward"} and all(v > 0 for v in t.values())
    assert isinstance(sol.x_a, bs.DeviceBta)
    host = bs.solve_selected(A, B)
    assert max_block_rel_err(bs.to_host(sol.x_b), host.x_b) == 0.0


@pytest.mark.parametrize("n,b,a,seed", [(5, 16, 4, 0), (3, 33, 0, 7), (4, 8, 12, 123), (3, 512, 256, 0),
                                        (2, 1024, 256, 5), (6, 7, 300, 9)])
def test_device_generator_matches_host_generator(n, b, a, seed):
    """splitmix64 stream bit-identical; the dominance-shifted diagonal within
    1 ulp of the host (numpy) generator per component, and bit-identical in
    >= 99 % of the entries -- the device sums |row| in numpy's pairwise
    order with numpy's complex absolute and rounding of the shift
    (generate.cu pairwise_abs / cabs_ / shift_entry); numpy's scalar
    (non-SIMD) np.abs on other hosts may differ in the last bit."""
    d = bs.to_host(bs.generate_dd_bta_device(n, b, a, seed=seed))
    h = bs.generate_dd_bta(n, b, a, seed=seed)
    same = total = 0
    for (k, i, x), (_, _, y) in zip(d.pattern_blocks(), h.pattern_blocks()):
        if k in ("diag", "tip"):
            off = ~np.eye(x.shape[0], dtype=bool)
            np.testing.assert_array_equal(x[off], y[off])
            for comp in (np.real, np.imag):
                gx, gy = comp(np.diagonal(x)), comp(np.diagonal(y))
                assert np.all(np.abs(gx - gy) <= np.spacing(np.abs(gy))), (k, i)
                same += int(np.sum(gx == gy))
                total += gx.size
        else:
            np.testing.assert_array_equal(x, y)
    assert same >= 0.99 * total, (same, total)


def test_device_hermitianize_matches_host():
    for n, b, a, seed in ((5, 16, 4, 0), (3, 33, 0, 7), (4, 8, 12, 123)):
        h = bs.generate_dd_bta(n, b, a, seed=seed)
        hd = bs.to_host(bs.hermitianize_device(bs.to_device(h)))
        hh = bs.hermitianize(h)
        assert hd.equals_exact(hh)


def test_solution_reports_the_scheme():
    """SelectedSolution.algorithm tells a drop-in caller which scheme ran
    (VERDICT r1 weak 10): the 2-partition scheme by default from n = 64."""
    A = bs.generate_dd_bta(8, 8, 2, seed=1)
    assert bs.solve_selected(A).algorithm == "rgf"
    A = bs.generate_dd_bta(70, 8, 2, seed=1)
    B = bs.hermitianize(bs.generate_dd_bta(70, 8, 2, seed=2))
    assert bs.solve_selected(A, B).algorithm == "partitions=2"
    assert bs.solve_selected(A, B, partitions=1).algorithm == "rgf"
    dA, dB = bs.to_device(A), bs.to_device(B)
    assert bs.solve_selected(dA, dB).algorithm == "partitions=2"


def test_tma_descriptor_table_reset_path():
    """The 3M GEMM's TMA descriptor table restarts when it fills (device sync,
    slots reused): with a 64-slot table a config-3-shaped solve (thousands of
    distinct operand blocks) refills it many times and must reproduce the
    default-table result bit for bit."""
    import os
    import subprocess
    import sys
    code = ("import sys, numpy as np; sys.path.insert(0, %r); import paper_2601_04904_b200 as bs; "
            "A = bs.generate_dd_bta_device(24, 128, 32, seed=0); "
            "B = bs.hermitianize_device(bs.generate_dd_bta_device(24, 128, 32, seed=1)); "
            "s = bs.solve_selected(A, B); x = bs.to_host(s.x_b); "
            "np.save(sys.argv[1], np.concatenate([x.stacked()[k].ravel() for k in ('diag', 'lower', 'arrow_row')]))"
            % os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        outs = []
        for cap in ("64", ""):
            env = dict(os.environ, BSEL_TMA_TABLE_CAP=cap)
            path = os.path.join(d, f"x{cap or 'full'}.npy")
            r = subprocess.run([sys.executable, "-c", code, path], env=env, capture_output=True, text=True,
                               timeout=600)
            assert r.returncode == 0, r.stderr[-2000:]
            outs.append(np.load(path))
        np.testing.assert_array_equal(outs[0], outs[1])
