"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and the reference's known-answer tests."""

import numpy as np
import pytest
from conftest import load_case, manifest, max_block_rel_err, quadratic_block_residual, identity_block_row_residual

import oracle
from oracle.seq import Blocks, _Mul, forward

M = manifest()
SEQ = sorted(k for k, v in M["cases"].items() if v["kind"] == "seq")
DIST = sorted(k for k, v in M["cases"].items() if v["kind"] == "dist")


def _inputs_match(meta, A, B):
    g = oracle.generate_dd_bta(meta["n"], meta["b"], meta["a"], seed=meta["seed"])
    for (_, _, x), (_, _, y) in zip(g.blocks(), A.blocks()):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("name", SEQ)
def test_oracle_matches_reference_seq(name):
    meta, A, B, XA, XB = load_case(name)
    _inputs_match(meta, A, B)
    counts = {}
    from collections import Counter
    c = Counter()
    xa, xb = oracle.solve_selected(A, B, meta["mode"], counts=c)
    assert max_block_rel_err(xa, XA) <= 1e-13
    if XB is not None:
        assert max_block_rel_err(xb, XB) <= 1e-13
    ref_counts = {k[5:]: v for k, v in meta["counts"].items() if k.startswith("gemm_")}
    assert dict(c) == ref_counts


@pytest.mark.parametrize("name", DIST)
def test_oracle_matches_reference_dist(name):
    meta, A, B, XA, XB = load_case(name)
    _inputs_match(meta, A, B)
    ranges, kinds = oracle.plan_partitions(meta["n"], meta["parts"], meta["mode"])
    assert [list(r) for r in ranges] == meta["ranges"]
    from collections import Counter
    c = Counter()
    log = []
    xa, xb = oracle.dist_solve(A, B, num_parts=meta["parts"], mode=meta["mode"], counts=c, payload_log=log)
    assert max_block_rel_err(xa, XA) <= 1e-13
    if XB is not None:
        assert max_block_rel_err(xb, XB) <= 1e-13
    ref_counts = {k[5:]: v for k, v in meta["counts"].items() if k.startswith("gemm_")}
    assert dict(c) == ref_counts
    gather = meta["trace"][0]
    assert gather["kind"] == "all_gather"
    for pay, ref in zip(log, gather["payloads"]):
        nbytes = sum(x.nbytes for key in ("diag", "arrow_row", "arrow_col", "coupling", "b_diag",
                                          "b_arrow_row", "b_arrow_col", "b_coupling")
                     for x in (pay.get(key) or []))
        assert nbytes == ref["nbytes"]


def test_generator_probe_and_config1_digest():
    p = M["generator_probe"]
    g = oracle.generate_dd_bta(p["n"], p["b"], p["a"], seed=p["seed"])
    np.testing.assert_array_equal(g.diag[0][0], [complex(*z) for z in p["diag0_row0"]])
    np.testing.assert_array_equal(g.tip, [[complex(*z) for z in row] for row in p["tip"]])
    a = oracle.generate_dd_bta(16, 64, 0, seed=0)
    xa, _ = oracle.solve_selected(a, None, "si")
    d = M["config1_digest"]
    norms = [np.linalg.norm(blk) for _, _, blk in xa.blocks() if blk.size]
    np.testing.assert_allclose(norms, d["norm"], rtol=1e-13)
    assert identity_block_row_residual(a, xa) <= 1e-13


def test_known_answers():
    k = M["known"]
    two = Blocks(2, 1, 0, [np.array([[2.0 + 0j]]), np.array([[2.0 + 0j]])], [np.array([[1.0 + 0j]])],
                 [np.array([[1.0 + 0j]])], [np.zeros((0, 1))] * 2, [np.zeros((1, 0))] * 2, np.zeros((0, 0)))
    mul = _Mul(1, 0)
    F = forward(Blocks.of(two), None, mul)
    np.testing.assert_allclose([s[0, 0] for s in F.s_a], k["two_block_s_a"])
    xa, _ = oracle.solve_selected(two)
    np.testing.assert_allclose(oracle.to_dense(xa), k["two_by_two_inverse"])
    arrow = Blocks(1, 1, 1, [np.array([[2.0 + 0j]])], [], [], [np.array([[1.0 + 0j]])], [np.array([[1.0 + 0j]])],
                   np.array([[3.0 + 0j]]))
    F = forward(Blocks.of(arrow), None, _Mul(1, 1))
    np.testing.assert_allclose(F.tip_inv, [[k["scalar_arrow_tip_schur_inv"]]])
    xa, _ = oracle.solve_selected(arrow)
    np.testing.assert_allclose(oracle.to_dense(xa), k["scalar_arrow_inverse"])


@pytest.mark.parametrize("key", sorted(M["op_counts"]))
def test_op_count_inventory(key):
    mode, n, a = key.split("_")
    n, a = int(n[1:]), int(a[1:])
    ref = M["op_counts"][key]
    tot, inv = oracle.op_counts(n, 8, a, mode)
    assert tot == {k[5:]: v for k, v in ref["total"].items() if k.startswith("gemm_")}
    assert inv == ref["total"]["inv"]
    fwd, _ = oracle.op_counts(n, 8, a, mode, forward_only=True)
    assert fwd == {k[5:]: v for k, v in ref["forward"].items() if k.startswith("gemm_")}


def test_dense_oracle_and_quadratic_residual():
    a = oracle.generate_dd_bta(6, 5, 3, seed=3)
    b = oracle.hermitianize(oracle.generate_dd_bta(6, 5, 3, seed=4))
    xa, xb = oracle.solve_selected(a, b)
    da, db = oracle.dense_selected(a, b)
    assert max_block_rel_err(xa, da) <= 1e-12
    assert max_block_rel_err(xb, db) <= 1e-12
    assert quadratic_block_residual(a, b, xa, xb) <= 1e-12


def test_singular_pivot_index():
    a = oracle.generate_dd_bta(4, 3, 0, seed=5)
    a.diag[2][:] = 0.0
    a.lower[1][:] = 0.0
    with pytest.raises(oracle.OracleSingular) as info:
        oracle.solve_selected(a)
    assert info.value.index == 2
