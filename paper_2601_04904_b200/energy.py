"""Energy-point sweep driver (SURVEY.md 8(e) "Energy sweep", 8(f)1; config 5).

A quantum-transport calculation solves one BTA system per energy point; the
points are independent.  Energy e is defined here by the bench protocol's
seeds: A_e = generate_dd_bta(n, b, a, seed=2e), B_e = hermitianize(
generate_dd_bta(n, b, a, seed=2e+1)) (energy 0 is config 4's bench system).
The reference has no energy concept; this is the driver the north star's
config 5 asks for.

One GPU: energies run back to back through ``solve_selected`` (two
concurrent in-GPU partitions each); the inputs of energy e+1 are generated
on a side stream into the second of two input buffers while energy e solves
(the generator is HBM-bound, the solve DMMA-bound).  Several GPUs: energy
parallel, energies e = rank, rank + world, ... on each rank, no collective
(weak scaling: fixed energies per GPU).
"""

from __future__ import annotations

import torch

from .device import DeviceBta, generate_dd_bta_device, hermitianize_device
from .rgf import default_partitions, solve_selected

__all__ = ["EnergySweep", "energy_seeds", "rank_energies"]


def energy_seeds(e: int) -> tuple[int, int]:
    """Generator seeds of energy point e (A, B)."""
    return 2 * e, 2 * e + 1


def rank_energies(energies, world: int, rank: int):
    """Energy-parallel assignment: round robin over ranks."""
    return [e for i, e in enumerate(energies) if i % world == rank]


class EnergySweep:
    """Solve many energy points of one shape on one GPU with preallocated
    buffers; ``run`` calls ``consume(e, solution)`` after each energy (the
    solution's device buffers are reused by the next energy)."""

    def __init__(self, n: int, b: int, a: int, mode: str = "siq", device=None, partitions=None,
                 dominance: float = 1.5):
        self.n, self.b, self.a, self.mode = n, b, a, mode
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.parts = default_partitions(n) if partitions is None else partitions
        self.dominance = dominance
        fused = mode == "siq"
        mk = lambda: DeviceBta.empty(n, b, a, self.device, zero=False)  # noqa: E731
        self.inputs = [(mk(), mk() if fused else None) for _ in range(2)]
        self.out = (mk(), mk() if fused else None)
        self.gen_stream = torch.cuda.Stream(self.device)
        self._free = [None, None]  # event: input slot no longer read by a solve

    def _generate(self, e: int, slot: int) -> torch.cuda.Event:
        A, B = self.inputs[slot]
        sa, sb = energy_seeds(e)
        with torch.cuda.device(self.device), torch.cuda.stream(self.gen_stream):
            if self._free[slot] is not None:
                self.gen_stream.wait_event(self._free[slot])
            generate_dd_bta_device(self.n, self.b, self.a, sa, self.dominance, out=A)
            if B is not None:
                hermitianize_device(generate_dd_bta_device(self.n, self.b, self.a, sb, self.dominance, out=B))
            ready = torch.cuda.Event()
            ready.record(self.gen_stream)
        return ready

    def run(self, energies, consume=None, timings=None):
        """Solve ``energies`` in order; returns the number solved."""
        energies = list(energies)
        if not energies:
            return 0
        main = torch.cuda.current_stream(self.device)
        ready = self._generate(energies[0], 0)
        for k, e in enumerate(energies):
            slot = k & 1
            if k + 1 < len(energies):  # overlap the next energy's inputs with this solve
                nxt = self._generate(energies[k + 1], slot ^ 1)
            main.wait_event(ready)
            A, B = self.inputs[slot]
            sol = solve_selected(A, B, self.mode, out=self.out, partitions=self.parts, timings=timings)
            done = torch.cuda.Event()
            done.record(main)
            self._free[slot] = done
            if consume is not None:
                consume(e, sol)
            if k + 1 < len(energies):
                ready = nxt
        return len(energies)
