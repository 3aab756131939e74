"""BTA1 streaming to / from the device."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200 import fileio  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("shape", [(1, 1, 0), (3, 2, 1), (7, 33, 5), (16, 64, 16)])
def test_device_roundtrip_bytewise(tmp_path, shape, monkeypatch):
    monkeypatch.setattr(fileio, "_STAGE_BYTES", 4096)  # many ragged staging chunks
    m = bs.generate_dd_bta(*shape, seed=7)
    host_file, dev_file = tmp_path / "h.bta", tmp_path / "d.bta"
    bs.write_bta(m, host_file)
    X = bs.read_bta_device(host_file)
    assert bs.to_host(X).equals_exact(m)
    bs.write_bta(X, dev_file)
    assert dev_file.read_bytes() == host_file.read_bytes()


def test_device_read_reference_file_and_errors(tmp_path):
    X = bs.read_bta_device(os.path.join(GOLDEN, "bta1_sol_xb_5_4_2.bta"))
    assert bs.to_host(X).equals_exact(bs.read_bta(os.path.join(GOLDEN, "bta1_sol_xb_5_4_2.bta")))
    m = bs.generate_dd_bta(2, 2, 1, seed=0)
    m.arrow_col[1][0, 0] = np.inf
    bs.write_bta(m, tmp_path / "bad.bta")
    with pytest.raises(bs.ShapeInconsistencyError):
        bs.read_bta_device(tmp_path / "bad.bta")
    raw = (tmp_path / "bad.bta").read_bytes()
    (tmp_path / "short.bta").write_bytes(raw[:-8])
    with pytest.raises(bs.TruncatedPayloadError):
        bs.read_bta_device(tmp_path / "short.bta")


def test_file_to_solution_to_file(tmp_path):
    """CLI-shaped flow: BTA1 in -> device solve -> BTA1 out, vs host solve."""
    A = bs.generate_dd_bta(6, 8, 3, seed=1)
    B = bs.hermitianize(bs.generate_dd_bta(6, 8, 3, seed=2))
    bs.write_bta(A, tmp_path / "a.bta")
    bs.write_bta(B, tmp_path / "b.bta")
    sol = bs.solve_selected(bs.read_bta_device(tmp_path / "a.bta"), bs.read_bta_device(tmp_path / "b.bta"), "siq")
    bs.write_bta(sol.x_b, tmp_path / "xb.bta")
    ref = bs.solve_selected(A, B, "siq")
    assert bs.read_bta(tmp_path / "xb.bta").equals_exact(ref.x_b)
