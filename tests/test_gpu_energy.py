"""Energy-point sweep driver (config 5 path)."""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04904_b200 as bs  # noqa: E402
from conftest import max_block_rel_err  # noqa: E402


@pytest.mark.parametrize("parts", [1, 2])
def test_sweep_matches_individual_solves(parts):
    n, b, a = 12, 16, 8
    sweep = bs.EnergySweep(n, b, a, "siq", partitions=parts)
    got = {}
    sweep.run([3, 0, 5], consume=lambda e, sol: got.__setitem__(e, (bs.to_host(sol.x_a), bs.to_host(sol.x_b))))
    assert sorted(got) == [0, 3, 5]
    for e, (xa, xb) in got.items():
        sa, sb = bs.energy_seeds(e)
        A = bs.generate_dd_bta_device(n, b, a, seed=sa)
        B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=sb))
        ref = bs.solve_selected(A, B, "siq", partitions=parts)
        assert xa.equals_exact(bs.to_host(ref.x_a)) and xb.equals_exact(bs.to_host(ref.x_b))


def test_energy_zero_is_the_bench_system_and_si_mode():
    sweep = bs.EnergySweep(6, 8, 0, "si", partitions=1)
    out = []
    sweep.run([0], consume=lambda e, sol: out.append(bs.to_host(sol.x_a)))
    ref = bs.solve_selected(bs.generate_dd_bta(6, 8, 0, seed=0), None, "si", partitions=1)
    assert out[0].equals_exact(ref.x_a) or max(
        float(abs(x - y).max()) for x, y in zip(out[0].diag, ref.x_a.diag)) < 1e-13


@pytest.mark.parametrize("out_slots,parts,mode", [(2, 2, "siq"), (1, 2, "siq"), (None, 2, "siq"), (2, 1, "siq"), (2, 1, "si")])
def test_host_sweep_matches_individual_solves(out_slots, parts, mode):
    """Pipelined host-buffer sweep: every energy's host outputs equal the
    single-call device solve bit for bit (4 energies: both input and output
    slots are reused)."""
    n, b, a = 10, 16, 8
    energies = [0, 1, 2, 3]
    ins, outs = [], []
    for e in energies:
        sa, sb = bs.energy_seeds(e)
        ha = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
        bs.generate_dd_bta_device(n, b, a, seed=sa).copy_to_host(ha)
        hb = None
        if mode == "siq":
            hb = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
            bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=sb)).copy_to_host(hb)
        ins.append((ha, hb))
        outs.append((bs.BtaMatrix.zeros(n, b, a, pinned=True),
                     bs.BtaMatrix.zeros(n, b, a, pinned=True) if mode == "siq" else None))
    sweep = bs.HostEnergySweep(n, b, a, mode, partitions=parts, out_slots=out_slots)
    assert sweep.run(ins, outs) == len(energies)
    for k, ((ha, hb), (xa, xb)) in enumerate(zip(ins, outs)):
        ref = bs.solve_selected(bs.to_device(ha), bs.to_device(hb) if hb is not None else None, mode,
                                partitions=parts)
        assert xa.equals_exact(bs.to_host(ref.x_a))
        if mode == "siq":
            if k == 0 and parts > 1:
                # energy 0 streams its pinned inputs in behind the forward:
                # X_B to rounding (see test_gpu_dist streamed host I/O)
                assert max_block_rel_err(xb, bs.to_host(ref.x_b)) <= 1e-13
            else:
                assert xb.equals_exact(bs.to_host(ref.x_b))


@pytest.mark.parametrize("parts", [1, 2])
def test_concurrent_energies_match_individual_solves(parts):
    """Two energies in flight (EnergySweep concurrent=2: own buffers, runners
    and lane contexts per pipe, host thread per pipe): every energy's solution
    bit-identical to its single solve."""
    n, b, a = 12, 16, 8
    sweep = bs.EnergySweep(n, b, a, "siq", partitions=parts, concurrent=2)
    assert sweep.concurrent == 2
    got = {}
    sweep.run([4, 1, 6, 2, 0], consume=lambda e, sol: got.__setitem__(
        e, (bs.to_host(sol.x_a), bs.to_host(sol.x_b))))
    torch.cuda.synchronize()
    assert sorted(got) == [0, 1, 2, 4, 6]
    for e, (xa, xb) in got.items():
        sa, sb = bs.energy_seeds(e)
        A = bs.generate_dd_bta_device(n, b, a, seed=sa)
        B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=sb))
        ref = bs.solve_selected(A, B, "siq", partitions=parts)
        assert xa.equals_exact(bs.to_host(ref.x_a)) and xb.equals_exact(bs.to_host(ref.x_b))


def test_overlapped_energies_match_individual_solves():
    """EnergySweep overlap: energy k+1's forward runs during energy k's
    backward (second partition runner, one output set); every energy's
    solution bit-identical to its single solve."""
    n, b, a = 70, 16, 8
    sweep = bs.EnergySweep(n, b, a, "siq", overlap=True)
    assert sweep.overlap
    got = {}
    sweep.run([3, 0, 5, 1, 2], consume=lambda e, sol: got.__setitem__(
        e, (bs.to_host(sol.x_a), bs.to_host(sol.x_b))))
    assert sorted(got) == [0, 1, 2, 3, 5]
    for e, (xa, xb) in got.items():
        sa, sb = bs.energy_seeds(e)
        A = bs.generate_dd_bta_device(n, b, a, seed=sa)
        B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=sb))
        ref = bs.solve_selected(A, B, "siq")
        assert xa.equals_exact(bs.to_host(ref.x_a)) and xb.equals_exact(bs.to_host(ref.x_b))
