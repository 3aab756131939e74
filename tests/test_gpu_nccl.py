"""Multi-GPU distributed solve over NCCL (one process per GPU), vs the oracle.
Needs >= 2 GPUs (gpurun --gpus 2|4); skipped otherwise."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, n, b, a, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        import oracle
        import paper_2601_04904_b200 as bs
        from conftest import max_block_rel_err
        A = bs.generate_dd_bta(n, b, a, seed=0)
        B = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=1))
        coll = bs.TorchCollectives()
        sol = bs.dist_solve(A, B, num_parts=world, mode="siq", transport=coll)
        kinds = [e.kind for e in coll.trace]
        err = None
        if rank == 0:
            xa, xb = oracle.dist_solve(A, B, num_parts=world, mode="siq")
            err = max(max_block_rel_err(sol.x_a, xa), max_block_rel_err(sol.x_b, xb))
        else:
            assert sol is None
        # bench path: DistSolver on device-generated inputs, sharded outputs
        dA = bs.generate_dd_bta_device(n, b, a, seed=0)
        dB = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1))
        s = bs.DistSolver(dA, dB, "siq", world, rank, torch.device("cuda", rank))
        s.solve()
        XA, XB = s.solve()
        # end-to-end path: host windows streamed behind the sweeps, bit-identical
        lo, hi = s.plan.ranges[rank]
        c = min(hi, n - 1)
        ref = [(X.diag[lo:hi].cpu(), X.arrow_row[lo:hi].cpu(), X.lower[lo:c].cpu(), X.upper[lo:c].cpu(),
                X.tip.cpu()) for X in (XA, XB)]
        seps = [s.plan.ranges[p][1] - 1 for p in range(world - 1)]
        win = tuple(bs.HostWindow(n, b, a, lo, hi, seps).fill_from(M) for M in (dA, dB))
        hout = (bs.HostWindow(n, b, a, lo, hi), bs.HostWindow(n, b, a, lo, hi))
        dA.diag.zero_()  # prove the streamed path does not read the device inputs' blocks
        dA.lower.zero_()
        os.environ["BSEL_STREAM_CHUNK"] = "3"
        for _ in range(2):
            s.solve(host_in=win, host_out=hout)
            torch.cuda.synchronize()
            # X_A bit-identical; X_B to rounding (the device-resident forward may
            # take the Hermitian-B path, streamed chunks cannot know it in advance)
            for side, (R, H) in enumerate(zip(ref, hout)):
                got = (H.diag, H.arrow_row, H.lower, H.upper) + ((H.tip,) if rank == 0 else ())
                for g_, r_ in zip(got, R):
                    if side == 0:
                        assert torch.equal(g_, r_)
                    elif r_.numel():
                        assert torch.linalg.norm(g_ - r_) <= 1e-12 * torch.linalg.norm(r_)
        # pipelined end-to-end form (DistSolver.solve_energies): 3 energies,
        # each one's owned outputs in its own host windows
        outs = [(bs.HostWindow(n, b, a, lo, hi), bs.HostWindow(n, b, a, lo, hi)) for _ in range(3)]
        s.solve_energies([win] * 3, outs)
        torch.cuda.synchronize()
        for H2 in outs:
            for side, (R, H) in enumerate(zip(ref, H2)):
                got = (H.diag, H.arrow_row, H.lower, H.upper) + ((H.tip,) if rank == 0 else ())
                for g_, r_ in zip(got, R):
                    if side == 0:
                        assert torch.equal(g_, r_)
                    elif r_.numel():
                        assert torch.linalg.norm(g_ - r_) <= 1e-12 * torch.linalg.norm(r_)
        dist.barrier()
        q.put((rank, err, kinds, None))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, None, None, traceback.format_exc()))


@pytest.mark.parametrize("world,n,b,a", [(2, 16, 64, 16), (2, 9, 40, 0), (4, 24, 48, 8)])
def test_nccl_dist_solve_matches_oracle(world, n, b, a):
    world = min(world, torch.cuda.device_count())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, n, b, a, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for rank, err, kinds, tb in res:
        assert tb is None, tb
        assert kinds == (["all_gather", "all_reduce"] if a else ["all_gather"])
    assert res[0][1] <= 1e-10


def _rank_k(rank, world, k, port, n, b, a, q):
    """k partitions per rank (DistSolver parts_per_rank): the world*k plan
    (e.g. the reference's 8-partition plan on 4 GPUs) vs the oracle, device
    path and host-window streaming path."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        import oracle
        import paper_2601_04904_b200 as bs
        from conftest import max_block_rel_err
        dA = bs.generate_dd_bta_device(n, b, a, seed=0)
        dB = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1))
        coll = bs.TorchCollectives()
        s = bs.DistSolver(dA, dB, "siq", world, rank, dev, transport=coll, parts_per_rank=k)
        XA, XB = s.solve()
        kinds = [e.kind for e in coll.trace]
        # merge the sharded outputs on rank 0 (disjoint blocks: exact sum)
        for m in (XA, XB):
            for t in m.tensors().values():
                if t.numel():
                    dist.reduce(torch.view_as_real(t), dst=0)
        err = None
        if rank == 0:
            A = bs.to_host(dA)
            B = bs.to_host(dB)
            xa, xb = oracle.dist_solve(A, B, num_parts=world * k, mode="siq")
            err = max(max_block_rel_err(bs.to_host(XA), xa), max_block_rel_err(bs.to_host(XB), xb))
        # host-window streaming over the union of this rank's partitions
        lo, hi = s.owned_range()
        seps = [s.plan.ranges[p][1] - 1 for p in range(world * k - 1)]
        win = tuple(bs.HostWindow(n, b, a, lo, hi, seps).fill_from(M) for M in (dA, dB))
        hout = (bs.HostWindow(n, b, a, lo, hi), bs.HostWindow(n, b, a, lo, hi))
        ref = s.solve()
        c = min(hi, n - 1)
        refc = [(X.diag[lo:hi].cpu(), X.lower[lo:c].cpu()) for X in ref]
        s.solve(host_in=win, host_out=hout)
        torch.cuda.synchronize()
        serr = 0.0
        for (rd, rl), H in zip(refc, hout):
            for g_, r_ in ((H.diag, rd), (H.lower, rl)):
                if r_.numel():
                    serr = max(serr, float(torch.linalg.norm(g_ - r_) / torch.linalg.norm(r_)))
        dist.barrier()
        q.put((rank, err, kinds, serr, None))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, None, None, None, traceback.format_exc()))


@pytest.mark.parametrize("world,k,n,b,a", [(2, 2, 20, 48, 8), (4, 2, 24, 32, 8), (4, 2, 40, 64, 16)])
def test_nccl_k_partitions_per_rank(world, k, n, b, a):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_k, args=(r, world, k, port, n, b, a, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for rank, err, kinds, serr, tb in res:
        assert tb is None, tb
        assert kinds == ["all_gather", "all_reduce"]  # one of each per solve, k partitions per rank
        assert serr <= 1e-12
    assert res[0][1] <= 1e-10


REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def _ref_rank(rank, world, port, n, b, a, q):
    """The reference's own dist.py per-rank pipeline driven over NCCL through
    TorchCollectives (numpy payloads as bytes), vs the reference's ThreadHub run."""
    try:
        import sys
        sys.path.insert(0, REF)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        import btasel
        from btasel import dist as rdist
        import paper_2601_04904_b200 as bs
        btasel.set_blas_threads(1)
        A = btasel.generate_dd_bta(n, b, a, seed=5)
        B = btasel.hermitianize(btasel.generate_dd_bta(n, b, a, seed=6))
        plan = btasel.plan_partitions(n, world, "siq")
        coll = bs.TorchCollectives()
        sl, _, _, _ = rdist._run_rank(A, B, plan, rank, coll, "siq", None)
        blobs = coll.gather_to_root(rdist._slice_to_bytes(sl))
        kinds = [e.kind for e in coll.trace]
        ok = None
        if rank == 0:
            got = rdist._merge_slices(A, "siq", [rdist._slice_from_bytes(x) for x in blobs])
            ref = btasel.dist_solve(A, B, num_parts=world, mode="siq")
            ok = got.x_a.equals_exact(ref.x_a) and got.x_b.equals_exact(ref.x_b)
        dist.barrier()
        q.put((rank, ok, kinds, None))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, None, None, traceback.format_exc()))


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "btasel")), reason="reference not staged")
@pytest.mark.parametrize("world,n,b,a", [(2, 10, 8, 4), (4, 24, 8, 4)])
def test_reference_dist_over_nccl(world, n, b, a):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ref_rank, args=(r, world, port, n, b, a, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for rank, ok, kinds, tb in res:
        assert tb is None, tb
        assert kinds[:2] == ["all_gather", "all_reduce"]  # + the output gather_to_root round
    assert res[0][1] is True


def _symm_rank(rank, world, port, n, b, a, q):
    """Boundary exchange by NVLink peer stores into symmetric memory
    (TorchCollectives(symmetric=True), bsel_publish) vs the NCCL all_gather:
    bit-identical solutions, one all_gather + one all_reduce per solve."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        import paper_2601_04904_b200 as bs
        dA = bs.generate_dd_bta_device(n, b, a, seed=0)
        dB = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1))
        ref = [t.clone() for X in bs.DistSolver(dA, dB, "siq", world, rank, dev).solve() for t in X.tensors().values()]
        coll = bs.TorchCollectives(symmetric=True)
        s = bs.DistSolver(dA, dB, "siq", world, rank, dev, transport=coll)
        for _ in range(3):  # the receive buffer is reused across solves
            got = [t for X in s.solve() for t in X.tensors().values()]
            torch.cuda.synchronize()
            same = all(torch.equal(x, y) for x, y in zip(got, ref))
        kinds = [e.kind for e in coll.trace]
        dist.barrier()
        q.put((rank, same, kinds, coll.exchange_impl, None))
        dist.destroy_process_group()
    except Exception:
        import traceback
        q.put((rank, None, None, None, traceback.format_exc()))


@pytest.mark.parametrize("world,n,b,a", [(2, 16, 64, 16), (4, 24, 48, 8)])
def test_symmetric_memory_exchange(world, n, b, a):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_symm_rank, args=(r, world, port, n, b, a, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for rank, same, kinds, impl, tb in res:
        assert tb is None, tb
        assert "bsel_publish" in impl, impl
        assert same
        assert kinds == ["all_gather", "all_reduce"] * 3
