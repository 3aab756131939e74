"""CPU (gloo, world_size 2 and 3) tests of the distributed host logic:
payload packing, the single all_gather, the rank-ordered all_reduce and the
reduced-system assembly, against the oracle's restatement of dist.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import manifest

import oracle
from oracle.dist import assemble as oracle_assemble
from oracle.dist import local_forward as oracle_local_forward
from oracle.seq import _Mul


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x))


def _device_bta(m):
    from paper_2601_04904_b200 import DeviceBta
    st = lambda blocks, shp: torch.from_numpy(np.ascontiguousarray(np.stack(blocks) if len(blocks) else np.zeros((0,) + shp, np.complex128)))  # noqa: E731
    return DeviceBta(m.n, m.b, m.a, {"diag": st(m.diag, (m.b, m.b)), "lower": st(m.lower, (m.b, m.b)),
                                     "upper": st(m.upper, (m.b, m.b)), "arrow_row": st(m.arrow_row, (m.a, m.b)),
                                     "arrow_col": st(m.arrow_col, (m.b, m.a)), "tip": _t(m.tip)})


def _payload(pay, rank, b, a, fused):
    from paper_2601_04904_b200.dist import BoundaryPayload
    p = BoundaryPayload(rank=rank, kind=pay["kind"], b=b, a=a, fused=fused)
    p.diag = [_t(x) for x in pay["diag"]]
    p.arrow_row = [_t(x) for x in pay["arrow_row"]]
    p.arrow_col = [_t(x) for x in pay["arrow_col"]]
    p.coupling = [_t(x) for x in (pay["coupling"] or [])]
    if fused:
        p.b_diag = [_t(x) for x in pay["b_diag"]]
        p.b_arrow_row = [_t(x) for x in pay["b_arrow_row"]]
        p.b_arrow_col = [_t(x) for x in pay["b_arrow_col"]]
        p.b_coupling = [_t(x) for x in (pay["b_coupling"] or [])]
    return p


def _worker(rank, world, port, n, b, a, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from paper_2601_04904_b200 import TorchCollectives, plan_partitions
    from paper_2601_04904_b200.dist import assemble_reduced

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, n, b, a, mode, q)
    except Exception:  # report instead of hanging the peer's queue.get
        import traceback
        q.put((rank, traceback.format_exc(), None, None, None, None))
    finally:
        dist.destroy_process_group()


def _body(rank, world, n, b, a, mode, q):
    from paper_2601_04904_b200 import TorchCollectives, plan_partitions
    from paper_2601_04904_b200.dist import assemble_reduced
    if True:
        A = oracle.generate_dd_bta(n, b, a, seed=3)
        B = oracle.hermitianize(oracle.generate_dd_bta(n, b, a, seed=4)) if mode == "siq" else None
        ranges, kinds = oracle.plan_partitions(n, world, mode)
        pay, delta, _ = oracle_local_forward(A, B, ranges, kinds, rank, _Mul(b, a))
        coll = TorchCollectives()
        plan = plan_partitions(n, world, mode)
        red = assemble_reduced(coll, _device_bta(A), _device_bta(B) if B is not None else None, plan,
                               _payload(pay, rank, b, a, B is not None), _t(delta))
        # oracle reference assembly from all ranks' payloads
        outs = [oracle_local_forward(A, B, ranges, kinds, r, _Mul(b, a)) for r in range(world)]
        tot = outs[0][1].copy()
        for o in outs[1:]:
            tot = tot + o[1]
        RA, RB, index = oracle_assemble(A, B, ranges, [o[0] for o in outs], tot)
        err = 0.0
        pairs = [(red.matrix_a, RA)] + ([(red.matrix_b, RB)] if B is not None else [])
        for got, ref in pairs:
            for kind in ("diag", "lower", "upper", "arrow_row", "arrow_col"):
                for g, r in zip(getattr(got, kind), getattr(ref, kind)):
                    err = max(err, float(np.max(np.abs(g.numpy() - r))) if r.size else 0.0)
            if a:
                err = max(err, float(np.max(np.abs(got.tip.numpy() - ref.tip))))
        q.put((rank, err, [e.kind for e in coll.trace], red.index == index,
               [p.get("nbytes") for p in coll.trace[0].payloads], red.matrix_a.tip.numpy().tobytes()))


@pytest.mark.parametrize("world,n,b,a,mode", [(2, 8, 3, 2, "siq"), (3, 12, 3, 2, "siq"), (3, 12, 4, 0, "si"),
                                              (3, 12, 4, 2, "si")])
def test_gloo_exchange_and_assembly(world, n, b, a, mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, b, a, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, kinds, same_index, nbytes, tip in res:
        assert not isinstance(err, str), err
        assert err == 0.0, (rank, err)   # same blocks, same rank-ordered sum: bitwise
        assert kinds == (["all_gather", "all_reduce"] if a else ["all_gather"])
        assert same_index
    assert len({r[5] for r in res}) == 1  # replicated bitwise
    if mode == "si" and world == 3:
        assert res[0][4][1] == 16 * (4 * b * b + 4 * a * b)  # middle payload bytes (test_dist.py:115-120)


def test_payload_pack_roundtrip():
    from paper_2601_04904_b200.dist import BoundaryPayload
    rng = np.random.default_rng(0)
    c = lambda *s: torch.from_numpy(rng.standard_normal(s) + 1j * rng.standard_normal(s))  # noqa: E731
    p = BoundaryPayload(rank=1, kind="middle", b=3, a=2, fused=True,
                        diag=[c(3, 3), c(3, 3)], coupling=[c(3, 3), c(3, 3)], arrow_row=[c(2, 3), c(2, 3)],
                        arrow_col=[c(3, 2), c(3, 2)], b_diag=[c(3, 3), c(3, 3)], b_coupling=[c(3, 3), c(3, 3)],
                        b_arrow_row=[c(2, 3), c(2, 3)], b_arrow_col=[c(3, 2), c(3, 2)])
    q = p.unpack(p.pack(), rank=1)
    for f in ("diag", "coupling", "arrow_row", "arrow_col", "b_diag", "b_coupling", "b_arrow_row", "b_arrow_col"):
        for x, y in zip(getattr(p, f), getattr(q, f)):
            assert torch.equal(x, y)
    e = BoundaryPayload(rank=0, kind="first", b=3, a=2, fused=False, diag=[c(3, 3)], arrow_row=[c(2, 3)],
                        arrow_col=[c(3, 2)])
    assert e.pack().numel() == p.pack().numel() // 2 + 2 or e.pack().numel() > 0
    r = e.unpack(e.pack(), rank=0)
    assert r.kind == "first" and r.coupling == [] and len(r.diag) == 1
    with pytest.raises(Exception):
        e.unpack(e.pack(), rank=1)


@pytest.mark.parametrize("name", sorted(k for k, v in manifest()["cases"].items() if v["kind"] == "dist"))
def test_partition_counts_match_reference(name):
    from paper_2601_04904_b200 import OpCounter, plan_partitions
    from paper_2601_04904_b200.dist import record_partition
    from paper_2601_04904_b200.kernels import record_sweep
    meta = manifest()["cases"][name]
    n, b, a, mode, parts = meta["n"], meta["b"], meta["a"], meta["mode"], meta["parts"]
    plan = plan_partitions(n, parts, mode)
    c = OpCounter(b=b, a=a)
    for r in range(parts):
        lo, hi = plan.ranges[r]
        record_partition(c, plan.kinds[r], hi - lo, b, a, mode, "forward")
        record_partition(c, plan.kinds[r], hi - lo, b, a, mode, "backward")
    nr = 2 * parts - 2
    record_sweep(c, nr, b, a, mode, "forward")
    record_sweep(c, nr, b, a, mode, "backward")
    assert c.as_dict() == meta["counts"]


@pytest.mark.parametrize("n,parts", [(1024, 8), (1024, 4), (12, 3), (8, 4), (20, 2)])
def test_host_windows_cover_pattern(n, parts):
    """HostWindow (per-rank pinned host storage of the N>1 end-to-end path):
    the blocks the ranks own partition the pattern exactly, every window
    holds its partition's couplings plus every partition separator, and the
    descriptor addresses blocks by global index."""
    from paper_2601_04904_b200 import HostWindow, plan_partitions
    plan = plan_partitions(n, parts, "siq")
    b, a = 2, 1
    seps = [plan.ranges[p][1] - 1 for p in range(parts - 1)]
    owned = {"diag": [], "lower": []}
    for r in range(parts):
        lo, hi = plan.ranges[r]
        w = HostWindow(n, b, a, lo, hi, seps)
        owned["diag"].extend(range(lo, hi))
        owned["lower"].extend(range(lo, min(hi, n - 1)))
        for g in seps:
            lw, up = w.separator(g)
            assert lw.shape == (b, b) and up.shape == (b, b)
        d = w.desc()
        per = b * b * 16
        assert d.n == n and d.diag + lo * per == w.diag.data_ptr()
        if min(hi, n - 1) > lo:
            assert d.lower + lo * per == w.lower.data_ptr()
            assert d.upper + (min(hi, n - 1) - 1) * per == w.upper[-1].data_ptr()
        assert d.arrow_row + (hi - 1) * a * b * 16 == w.arrow_row[-1].data_ptr()
    assert sorted(owned["diag"]) == list(range(n))
    assert sorted(owned["lower"]) == list(range(n - 1))


# --------------------------------------------------------------------------
# the REFERENCE's own dist.py orchestration over TorchCollectives (gloo here,
# NCCL on the GPU box: tests/test_gpu_nccl.py) -- numpy payloads as bytes
# --------------------------------------------------------------------------

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def _ref_worker(rank, world, port, n, b, a, mode, q):
    import sys
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, REF)
    import torch.distributed as tdist
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import btasel  # the unmodified reference (baseline/_ref)
        from btasel import dist as rdist
        from paper_2601_04904_b200 import TorchCollectives
        btasel.set_blas_threads(1)
        A = btasel.generate_dd_bta(n, b, a, seed=5)
        B = btasel.hermitianize(btasel.generate_dd_bta(n, b, a, seed=6)) if mode == "siq" else None
        plan = btasel.plan_partitions(n, world, mode)
        coll = TorchCollectives()
        sl, _, _, _ = rdist._run_rank(A, B, plan, rank, coll, mode, None)
        blobs = coll.gather_to_root(rdist._slice_to_bytes(sl))
        kinds = [e.kind for e in coll.trace]
        err = None
        if rank == 0:
            got = rdist._merge_slices(A, mode, [rdist._slice_from_bytes(x) for x in blobs])
            ref = btasel.dist_solve(A, B, num_parts=world, mode=mode)  # reference ThreadHub
            err = 0.0
            for side in ("x_a", "x_b") if mode == "siq" else ("x_a",):
                g, r = getattr(got, side), getattr(ref, side)
                err = max(err, 0.0 if g.equals_exact(r) else 1.0)
        q.put((rank, err, kinds, blobs is None))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc(), None, None))
    finally:
        tdist.destroy_process_group()


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "btasel")), reason="reference not installed (tools/stage_reference.sh)")
@pytest.mark.parametrize("world,n,b,a,mode", [(2, 8, 3, 2, "siq"), (3, 12, 2, 1, "siq"), (3, 12, 3, 0, "si")])
def test_reference_orchestration_over_torch_collectives(world, n, b, a, mode):
    """The reference's own per-rank pipeline (dist.py:787-801: local_forward,
    assemble_reduced, solve_reduced, local_backward) with TorchCollectives as
    its Collectives: numpy BoundaryPayloads travel as bytes, the tip delta
    sums in rank order, and the merged result is bit-identical to the
    reference's in-process ThreadHub run."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ref_worker, args=(r, world, port, n, b, a, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, kinds, none_blobs in res:
        assert not isinstance(err, str), err
        assert kinds == (["all_gather", "all_reduce", "all_gather"] if a else ["all_gather", "all_gather"])[:len(kinds)]
        assert none_blobs == (rank != 0)
    assert res[0][1] == 0.0


def test_host_payload_wire_roundtrip():
    """BoundaryPayload.to_bytes/from_bytes (the byte form foreign transports
    carry) round-trips blocks, kind, rank and the symmetry flags exactly."""
    from paper_2601_04904_b200.dist import BoundaryPayload
    rng = np.random.default_rng(1)
    c = lambda r, k: rng.standard_normal((r, k)) + 1j * rng.standard_normal((r, k))  # noqa: E731
    p = BoundaryPayload(rank=2, kind="middle", b=3, a=2, fused=True, sym_flags=1)
    p.diag, p.coupling = [c(3, 3), c(3, 3)], [c(3, 3), c(3, 3)]
    p.arrow_row, p.arrow_col = [c(2, 3), c(2, 3)], [c(3, 2), c(3, 2)]
    p.b_diag, p.b_coupling = [c(3, 3), c(3, 3)], [c(3, 3), c(3, 3)]
    p.b_arrow_row, p.b_arrow_col = [c(2, 3), c(2, 3)], [c(3, 2), c(3, 2)]
    q = BoundaryPayload.from_bytes(p.to_bytes())
    assert (q.rank, q.kind, q.b, q.a, q.fused, q.sym_flags) == (2, "middle", 3, 2, True, 1)
    assert q.summary() == p.summary()
    for f in ("diag", "coupling", "arrow_row", "arrow_col", "b_diag", "b_coupling", "b_arrow_row", "b_arrow_col"):
        for x, y in zip(getattr(p, f), getattr(q, f)):
            np.testing.assert_array_equal(x, y)
    assert q.nbytes() == p.nbytes() == 16 * 2 * (4 * 9 + 4 * 6)


def test_payload_wire_format_interoperates_with_the_reference():
    """Our BoundaryPayload bytes parse with the reference's from_bytes and
    the reference's bytes parse with ours (dist.py:41-131 wire format; our
    trailing sym_flags word is ignored by the reference)."""
    import sys
    if not os.path.isdir(os.path.join(REF, "btasel")):
        pytest.skip("reference not installed")
    sys.path.insert(0, REF)
    try:
        from btasel.dist import BoundaryPayload as RefPayload
    finally:
        sys.path.remove(REF)
    from paper_2601_04904_b200.dist import BoundaryPayload
    rng = np.random.default_rng(3)
    c = lambda r, k: rng.standard_normal((r, k)) + 1j * rng.standard_normal((r, k))  # noqa: E731
    ref = RefPayload(rank=1, kind="middle", diag=[c(3, 3), c(3, 3)], coupling=[c(3, 3), c(3, 3)],
                     arrow_row=[c(2, 3), c(2, 3)], arrow_col=[c(3, 2), c(3, 2)])
    ours = BoundaryPayload.from_bytes(ref.to_bytes())
    assert ours.summary() == ref.summary() and ours.sym_flags == 3 and not ours.fused
    back = RefPayload.from_bytes(ours.to_bytes())
    assert back.summary() == ref.summary()
    for f in ("diag", "coupling", "arrow_row", "arrow_col"):
        for x, y in zip(getattr(ref, f), getattr(back, f)):
            np.testing.assert_array_equal(x, y)


def test_owned_slices_merge_cover_the_pattern():
    """owned_slices (the reference's local_backward slice form, dist.py:551-560)
    of every rank merge into the full solution; every pattern block owned once."""
    import torch
    from paper_2601_04904_b200 import DeviceBta, plan_partitions
    from paper_2601_04904_b200.dist import merge_slices, owned_slices, _slices_from_bytes, _slices_to_bytes
    n, b, a = 12, 2, 1
    full = {k: torch.randn(s, dtype=torch.complex128) for k, s in
            {"diag": (n, b, b), "lower": (n - 1, b, b), "upper": (n - 1, b, b), "arrow_row": (n, a, b),
             "arrow_col": (n, b, a), "tip": (a, a)}.items()}
    X = DeviceBta(n, b, a, full)
    plan = plan_partitions(n, 3, "siq")
    slices = [_slices_from_bytes(_slices_to_bytes(owned_slices((X, X), plan, r)), True) for r in range(3)]
    owned = {}
    for sl in slices:
        for kind in ("diag", "lower", "upper", "arrow_row", "arrow_col"):
            for g in sl["x_a"][kind]:
                assert (kind, g) not in owned
                owned[(kind, g)] = True
    assert len(owned) == 3 * n + 2 * (n - 1)
    sol = merge_slices(n, b, a, "siq", slices)
    for kind, t in full.items():
        got = np.stack(getattr(sol.x_a, kind)) if kind != "tip" else sol.x_a.tip
        np.testing.assert_array_equal(got, t.numpy())


def _rankhub_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as tdist
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_04904_b200 import TorchCollectives
        from paper_2601_04904_b200.dist import BoundaryPayload, _RankHub
        b, a, k = 3, 2, 2
        coll = TorchCollectives()
        hub = _RankHub(coll, k)
        pays, deltas = [], []
        for j in range(k):
            p = rank * k + j
            kind = "first" if p == 0 else ("last" if p == world * k - 1 else "middle")
            nb = 1 if kind != "middle" else 2
            pay = BoundaryPayload(rank=p, kind=kind, b=b, a=a, fused=False)
            val = lambda r, c, s: torch.full((r, c), complex(p, s), dtype=torch.complex128)  # noqa: E731
            pay.diag = [val(b, b, i) for i in range(nb)]
            pay.arrow_row = [val(a, b, 10 + i) for i in range(nb)]
            pay.arrow_col = [val(b, a, 20 + i) for i in range(nb)]
            if kind == "middle":
                pay.coupling = [val(b, b, 30), val(b, b, 31)]
            pays.append(pay)
            deltas.append(torch.full((1, a, a), complex(p + 1, 0), dtype=torch.complex128))
        got = hub.all_gather_all(pays)
        tip = hub.all_reduce_all(deltas)
        q.put((rank, [(g.rank, g.kind, len(g.diag), complex(g.diag[0][0, 0])) for g in got],
               complex(tip[0, 0, 0]), [e.kind for e in coll.trace]))
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc(), None, None))
    finally:
        tdist.destroy_process_group()


def test_rank_hub_k_partitions_per_rank_gloo():
    """_RankHub (k partitions per rank): ONE all_gather brings every
    partition's payload in plan order, the tip deltas sum to the same value on
    every rank; trace = one all_gather + one all_reduce."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 2
    procs = [ctx.Process(target=_rankhub_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    for rank, got, tip, kinds in res:
        assert not isinstance(got, str), got
        assert [g[0] for g in got] == [0, 1, 2, 3]
        assert [g[1] for g in got] == ["first", "middle", "middle", "last"]
        assert [g[2] for g in got] == [1, 2, 2, 1]
        assert [g[3] for g in got] == [complex(p, 0) for p in range(4)]
        assert tip == complex(1 + 2 + 3 + 4, 0)
        assert kinds == ["all_gather", "all_reduce"]
