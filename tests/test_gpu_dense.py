"""GPU dense oracle (reference tests/test_baselines.py TestDenseSolve)."""

import numpy as np
import pytest
from conftest import max_block_rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2601_04904_b200 as bs  # noqa: E402


def _system(n, b, a, seed):
    return bs.generate_dd_bta(n, b, a, seed=seed), bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=seed + 1))


def test_identity_and_analytic():
    I = bs.BtaMatrix.identity(3, 2, 1)
    B = bs.generate_dd_bta(3, 2, 1, seed=0)
    sol = bs.dense_solve(I, B, "siq")
    assert max_block_rel_err(sol.x_b, B) <= 1e-14
    assert max_block_rel_err(sol.x_a, I) <= 1e-15


@pytest.mark.parametrize("n,b,a", [(5, 3, 2), (4, 16, 8), (1, 7, 3), (6, 5, 0)])
def test_matches_oracle_dense(n, b, a):
    A, B = _system(n, b, a, seed=2)
    sol = bs.dense_solve(A, B, "siq")
    xa, xb = oracle.dense_selected(A, B)
    assert max_block_rel_err(sol.x_a, xa) <= 1e-12
    assert max_block_rel_err(sol.x_b, xb) <= 1e-12


def test_cross_checks_rgf_at_mid_size():
    """N = 2112: dense GPU oracle vs the RGF sweeps (both on the GPU)."""
    A = bs.generate_dd_bta_device(8, 256, 64, seed=3)
    B = bs.hermitianize_device(bs.generate_dd_bta_device(8, 256, 64, seed=4))
    cnt = bs.OpCounter(b=256, a=64)
    d = bs.dense_solve(A, B, "siq", counter=cnt)
    assert isinstance(d.x_a, bs.DeviceBta)
    r = bs.solve_selected(A, B, "siq")
    assert max_block_rel_err(bs.to_host(d.x_a), bs.to_host(r.x_a)) <= 1e-10
    assert max_block_rel_err(bs.to_host(d.x_b), bs.to_host(r.x_b)) <= 1e-10
    assert cnt.lu_count == 1 and cnt.trsm_count == 2 and sum(cnt.gemm_by_shape.values()) == 2


def test_guard_and_si_mode():
    A = bs.generate_dd_bta(3, 2, 0, seed=3)
    with pytest.raises(bs.DenseGuardError):
        bs.dense_solve(A, guard=5)
    sol = bs.dense_solve(bs.generate_dd_bta(3, 2, 1, seed=4))
    assert sol.x_b is None and sol.mode == "si"
    with pytest.raises(ValueError):
        bs.dense_solve(A, None, "siq")
