"""Energy-point sweep driver (config 5 path)."""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2601_04904_b200 as bs  # noqa: E402


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
