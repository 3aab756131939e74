"""GPU tests of the distributed scheme (partition kernels + reduced system),
all partitions on one GPU through LocalHub; mirrors reference
tests/test_dist.py.  Multi-GPU NCCL runs: tests/test_gpu_nccl.py."""

import numpy as np
import pytest
from conftest import load_case, manifest, max_block_rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2601_04904_b200 as bs  # noqa: E402

M = manifest()
DIST = sorted(k for k, v in M["cases"].items() if v["kind"] == "dist")


def _bs(m):
    return bs.BtaMatrix(m.n, m.b, m.a, m.diag, m.lower, m.upper, m.arrow_row, m.arrow_col, m.tip)


def random_system(n, b, a, seed, hermitian_rhs=False):
    A = bs.generate_dd_bta(n, b, a, seed=seed)
    B = bs.generate_dd_bta(n, b, a, seed=seed + 1_000_003)
    return A, (bs.hermitianize(B) if hermitian_rhs else B)


@pytest.mark.parametrize("name", DIST)
def test_dist_vs_reference_golden(name):
    meta, A, B, XA, XB = load_case(name)
    cnt = bs.OpCounter(b=A.b, a=A.a)
    hub = bs.LocalHub(meta["parts"])
    sol = bs.dist_solve(_bs(A), _bs(B) if B is not None else None, num_parts=meta["parts"], mode=meta["mode"],
                        transport=hub, counter=cnt)
    assert max_block_rel_err(sol.x_a, XA) <= 1e-10
    if XB is not None:
        assert max_block_rel_err(sol.x_b, XB) <= 1e-10
    assert cnt.as_dict() == meta["counts"]
    assert [e.kind for e in hub.trace] == [t["kind"] for t in meta["trace"]]
    assert [p["nbytes"] for p in hub.trace[0].payloads] == [p["nbytes"] for p in meta["trace"][0]["payloads"]]


def _dist_vs_seq(n, b, a, parts, mode, seed=0, tol=1e-9):
    A, B = random_system(n, b, a, seed)
    B = B if mode == "siq" else None
    seq = bs.solve_selected(A, B, mode)
    got = bs.dist_solve(A, B, num_parts=parts, mode=mode)
    err = max_block_rel_err(got.x_a, seq.x_a)
    if mode == "siq":
        err = max(err, max_block_rel_err(got.x_b, seq.x_b))
    assert err <= tol, (n, b, a, parts, mode, err)


@pytest.mark.parametrize("parts", [2, 3, 4])
@pytest.mark.parametrize("mode", ["si", "siq"])
@pytest.mark.parametrize("a", [0, 2])
def test_matches_sequential(parts, mode, a):
    _dist_vs_seq(12, 3, a, parts, mode)


def test_eight_parts_and_minimum_partitions():
    _dist_vs_seq(20, 2, 1, 8, "siq")
    _dist_vs_seq(16, 3, 2, 8, "siq")
    _dist_vs_seq(8, 2, 0, 4, "si")
    _dist_vs_seq(4, 1, 0, 2, "si", tol=1e-12)


@pytest.mark.parametrize("n,b,a,parts", [(64, 64, 16, 4), (24, 128, 32, 4), (40, 96, 40, 8), (18, 200, 0, 3)])
def test_dist_vs_oracle_dist_larger_blocks(n, b, a, parts):
    A = bs.generate_dd_bta(n, b, a, seed=22)
    B = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=23))
    got = bs.dist_solve(A, B, num_parts=parts, mode="siq")
    xa, xb = oracle.dist_solve(A, B, num_parts=parts, mode="siq")
    assert max_block_rel_err(got.x_a, xa) <= 1e-10
    assert max_block_rel_err(got.x_b, xb) <= 1e-10


def test_single_part_bitwise_and_rerun_determinism():
    A, B = random_system(6, 3, 2, seed=1)
    seq = bs.solve_selected(A, B, "siq")
    got = bs.dist_solve(A, B, num_parts=1, mode="siq")
    assert got.x_a.equals_exact(seq.x_a) and got.x_b.equals_exact(seq.x_b)
    A, B = random_system(14, 3, 2, seed=2)
    s1 = bs.dist_solve(A, B, num_parts=4, mode="siq")
    s2 = bs.dist_solve(A, B, num_parts=4, mode="siq")
    assert s1.x_a.equals_exact(s2.x_a) and s1.x_b.equals_exact(s2.x_b)


def test_communication_contract():
    A, B = random_system(12, 3, 2, seed=3)
    hub = bs.LocalHub(3)
    bs.dist_solve(A, B, num_parts=3, mode="siq", transport=hub)
    assert [e.kind for e in hub.trace] == ["all_gather", "all_reduce"]
    middle = hub.trace[0].payloads[1]
    assert middle["kind"] == "middle"
    for side in ("", "b_"):
        assert middle["blocks"][side + "diag"] == [(3, 3), (3, 3)]
        assert middle["blocks"][side + "coupling"] == [(3, 3), (3, 3)]
    assert hub.trace[1].payloads[0]["elements"] == 2 * 2 * 2
    A0, _ = random_system(12, 4, 0, seed=4)
    hub = bs.LocalHub(3)
    bs.dist_solve(A0, num_parts=3, mode="si", transport=hub)
    assert [e.kind for e in hub.trace] == ["all_gather"]
    A2, _ = random_system(12, 4, 2, seed=6)
    hub = bs.LocalHub(3)
    bs.dist_solve(A2, num_parts=3, mode="si", transport=hub)
    assert hub.trace[0].payloads[1]["nbytes"] == 16 * (4 * 4 * 4 + 4 * 2 * 4)
    assert hub.trace[1].payloads[0]["elements"] == 2 * 2


def test_worker_error_carries_rank():
    A, _ = random_system(8, 2, 0, seed=14)
    A.diag[7][:] = 0.0
    with pytest.raises(bs.WorkerError) as info:
        bs.dist_solve(A, num_parts=2, mode="si")
    assert info.value.rank == 1
    assert isinstance(info.value.cause, bs.SingularBlockError) and info.value.cause.index == 7


def test_recursive_reduced_solve_timings_counters():
    A, B = random_system(24, 2, 1, seed=15)
    seq = bs.solve_selected(A, B, "siq")
    got = bs.dist_solve(A, B, num_parts=6, mode="siq", recursive_parts=2)
    assert max_block_rel_err(got.x_a, seq.x_a) <= 1e-9
    assert max_block_rel_err(got.x_b, seq.x_b) <= 1e-9
    t, cnt, per = {}, bs.OpCounter(b=3, a=2), []
    A, B = random_system(12, 3, 2, seed=16)
    bs.dist_solve(A, B, num_parts=3, mode="siq", timings=t, counter=cnt, rank_counters=per)
    assert set(t) == {"forward", "communication", "reduced", "backward"}
    assert len(per) == 3 and cnt.gemm_by_shape["bbb"] > sum(c.gemm_by_shape["bbb"] for c in per)


def test_identity_and_local_forward_payloads():
    sol = bs.dist_solve(bs.BtaMatrix.identity(12, 2, 2), num_parts=3, mode="si")
    assert max_block_rel_err(sol.x_a, bs.BtaMatrix.identity(12, 2, 2)) <= 1e-14
    A, _ = random_system(8, 2, 1, seed=8)
    plan = bs.plan_partitions(8, 2, "si")
    for rank in range(2):
        pay, _, _ = bs.local_forward(A, None, plan, rank)
        assert pay.coupling == [] and len(pay.diag) == 1
    A, _ = random_system(8, 2, 1, seed=9)
    plan = bs.plan_partitions(8, 4, "si")
    lo, hi = plan.ranges[1]
    assert hi - lo == 2
    pay, delta, fac = bs.local_forward(A, None, plan, 1)
    np.testing.assert_array_equal(np.asarray(pay.diag[0]), A.diag[lo])
    np.testing.assert_array_equal(pay.coupling[0], A.upper[lo])
    np.testing.assert_array_equal(pay.coupling[1], A.lower[lo])
    assert isinstance(delta, np.ndarray) and np.all(delta == 0)  # host in -> host out (dist.py:172-178)
    assert not fac.s_a  # nothing eliminated in a length-2 middle partition


def test_dist_device_inputs_stay_on_device():
    A = bs.generate_dd_bta_device(20, 32, 8, seed=0)
    B = bs.hermitianize_device(bs.generate_dd_bta_device(20, 32, 8, seed=1))
    got = bs.dist_solve(A, B, num_parts=4, mode="siq")
    assert isinstance(got.x_a, bs.DeviceBta)
    seq = bs.solve_selected(A, B, "siq")
    assert max_block_rel_err(bs.to_host(got.x_b), bs.to_host(seq.x_b)) <= 1e-9


@pytest.mark.parametrize("n,b,a,mode", [(64, 32, 16, "siq"), (70, 24, 0, "siq"), (66, 16, 8, "si"), (9, 8, 4, "siq")])
def test_solve_selected_partitions_match_sequential(n, b, a, mode):
    """solve_selected(partitions=2): the 2-partition scheme run concurrently
    on one GPU agrees with the sequential sweeps (and the oracle)."""
    A = bs.generate_dd_bta(n, b, a, seed=5)
    B = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=6)) if mode == "siq" else None
    seq = bs.solve_selected(A, B, mode, partitions=1)
    par = bs.solve_selected(A, B, mode, partitions=2)
    assert max_block_rel_err(par.x_a, seq.x_a) <= 1e-12
    if mode == "siq":
        assert max_block_rel_err(par.x_b, seq.x_b) <= 1e-12
    cnt1, cnt2 = bs.OpCounter(b=b, a=a), bs.OpCounter(b=b, a=a)
    t = {}
    bs.solve_selected(A, B, mode, partitions=1, counter=cnt1)
    d = bs.solve_selected(A, B, mode, partitions=2, counter=cnt2, timings=t, diagonal_only=True)
    assert cnt1.as_dict() == cnt2.as_dict() and set(t) == {"forward", "backward"}
    assert all(np.all(blk == 0) for blk in d.x_a.lower)


@pytest.mark.parametrize("parts,chunk", [(2, 3), (3, 2), (4, 1), (2, 64), (5, 4)])
@pytest.mark.parametrize("mode", ["si", "siq"])
def test_streamed_host_io_matches_device_path(parts, chunk, mode, monkeypatch):
    """Pinned host inputs/outputs streamed chunk by chunk behind the partition
    sweeps (bsel_host_io_t) give the results of device-resident inputs, for
    first/middle/last partitions and ragged chunk tails: X_A bit-identical;
    X_B to rounding (device-resident Hermitian B lets the forward skip the
    mirrored B-side products, which streamed chunks cannot know in advance)."""
    monkeypatch.setenv("BSEL_STREAM_CHUNK", str(chunk))
    n, b, a = 23, 8, 3
    A = bs.generate_dd_bta(n, b, a, seed=31, pinned=True)
    B = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=32)).copy(pinned=True) if mode == "siq" else None
    dev = bs.solve_selected(bs.to_device(A), bs.to_device(B) if B is not None else None, mode, partitions=parts)
    want_a, want_b = bs.to_host(dev.x_a), bs.to_host(dev.x_b) if mode == "siq" else None
    pinned_out = lambda: (bs.BtaMatrix.zeros(n, b, a, pinned=True), bs.BtaMatrix.zeros(n, b, a, pinned=True))  # noqa
    for inp, out in (((A, B), None), ((A, B), pinned_out()), ((A.copy(), B.copy() if B else None), pinned_out())):
        for _ in range(2):  # repeated solves reuse the runner's buffers
            got = bs.solve_selected(inp[0], inp[1], mode, partitions=parts, out=out)
            assert got.x_a.equals_exact(want_a)
            if mode == "siq":
                assert max_block_rel_err(got.x_b, want_b) <= 1e-13
    seq = bs.solve_selected(A, B, mode, partitions=1)
    assert max_block_rel_err(got.x_a, seq.x_a) <= 1e-12
