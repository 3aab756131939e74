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

import os

import torch

from .device import DeviceBta, generate_dd_bta_device, hermitianize_device
from .rgf import default_partitions, solve_selected

__all__ = ["EnergySweep", "HostEnergySweep", "energy_seeds", "rank_energies"]


def energy_seeds(e: int) -> tuple[int, int]:
    """Generator seeds of energy point e (A, B)."""
    return 2 * e, 2 * e + 1


def rank_energies(energies, world: int, rank: int):
    """Energy-parallel assignment: round robin over ranks."""
    return [e for i, e in enumerate(energies) if i % world == rank]


class EnergySweep:
    """Solve many energy points of one shape on one GPU with preallocated
    buffers; ``run`` calls ``consume(e, solution)`` after each energy (the
    solution's device buffers are reused by that pipe's next energy).

    Two energies in flight, two ways.  The forward sweeps are bound by their
    Schur chains (latency), the backward sweeps by the tensor pipe
    (throughput), so a second energy fills the SMs the first one's chains
    leave idle:

    * ``overlap`` (default when it fits: config 5 needs ~163 GB): energy
      k+1's forward runs while energy k's backward does, on a second
      partition runner, with ONE output set (``_run_overlapped``);
    * ``concurrent`` = k independent pipes, each with its own input / output
      buffers, partition runner and lane contexts, in its own host thread on
      its own streams (energies round robin); needs k full solve footprints,
      so it only fits for small shapes.

    Otherwise energies solve back to back and the next energy's inputs are
    generated on a side stream while the current one solves."""

    def __init__(self, n: int, b: int, a: int, mode: str = "siq", device=None, partitions=None,
                 dominance: float = 1.5, concurrent: int = 1, overlap: bool | None = None):
        self.n, self.b, self.a, self.mode = n, b, a, mode
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.parts = default_partitions(n) if partitions is None else partitions
        self.dominance = dominance
        fused = mode == "siq"
        self.concurrent = int(concurrent)
        # overlap: the next energy's forward runs while this energy's backward
        # does (second partition runner); default when the buffers fit
        if overlap is None:
            overlap = self.concurrent == 1 and self.parts > 1 and n >= 2 * self.parts and self._fits_overlap()
        self.overlap = bool(overlap) and self.parts > 1 and n >= 2 * self.parts
        self._runners = None
        mk = lambda: DeviceBta.empty(n, b, a, self.device, zero=False)  # noqa: E731
        # one pipe: two input slots (generation overlapped with the solve);
        # several pipes: one input slot each (the other pipe's solve overlaps it)
        nin = 2 if self.concurrent == 1 else 1
        self.pipes = []
        for _ in range(self.concurrent):
            self.pipes.append({"inputs": [(mk(), mk() if fused else None) for _ in range(nin)],
                               "out": (mk(), mk() if fused else None),
                               "gen": torch.cuda.Stream(self.device), "stream": torch.cuda.Stream(self.device),
                               "free": [None] * nin})
        # single-pipe aliases (round-1 attribute names)
        self.inputs, self.out = self.pipes[0]["inputs"], self.pipes[0]["out"]
        self.gen_stream = self.pipes[0]["gen"]

    def _bytes(self):
        """(one BTA matrix, one partition runner's factors + working strips)."""
        n, b, a = self.n, self.b, self.a
        blocks = 16 * (n * b * b + 2 * (n - 1) * b * b + 2 * n * a * b + a * a)
        fac = 16 * n * (7 * b * b + 6 * a * b)
        return blocks, fac

    def _fits_overlap(self) -> bool:
        """Device memory for the overlapped form: this sweep's two input slots
        and one output set (allocated below) + a second partition runner."""
        blocks, fac = self._bytes()
        free, _ = torch.cuda.mem_get_info(self.device)
        return (6 * blocks + 2 * fac) * 1.05 < free

    def _generate(self, pipe, e: int, slot: int) -> torch.cuda.Event:
        A, B = pipe["inputs"][slot]
        sa, sb = energy_seeds(e)
        g = pipe["gen"]
        with torch.cuda.device(self.device), torch.cuda.stream(g):
            if pipe["free"][slot] is not None:
                g.wait_event(pipe["free"][slot])
            # a generator context of this pipe: with concurrent pipes (host
            # threads), the default context is pipe 0's solve context, whose
            # stream binding another thread must not change mid-solve
            lane = 0 if self.concurrent == 1 else 2000 + self.pipes.index(pipe)
            generate_dd_bta_device(self.n, self.b, self.a, sa, self.dominance, out=A, _lane=lane)
            if B is not None:
                hermitianize_device(generate_dd_bta_device(self.n, self.b, self.a, sb, self.dominance, out=B,
                                                           _lane=lane), _lane=lane)
            ready = torch.cuda.Event()
            ready.record(g)
        return ready

    def _run_pipe(self, p: int, energies, consume, timings, lock):
        pipe = self.pipes[p]
        nin = len(pipe["inputs"])
        main = pipe["stream"]
        with torch.cuda.device(self.device), torch.cuda.stream(main):
            main.wait_stream(self._caller)
            ready = self._generate(pipe, energies[0], 0)
            for k, e in enumerate(energies):
                slot = k % nin
                nxt = None
                if k + 1 < len(energies) and nin > 1:  # overlap the next energy's inputs with this solve
                    nxt = self._generate(pipe, energies[k + 1], (k + 1) % nin)
                main.wait_event(ready)
                A, B = pipe["inputs"][slot]
                sol = solve_selected(A, B, self.mode, out=pipe["out"], partitions=self.parts, timings=timings,
                                     _pipe=p)
                done = torch.cuda.Event()
                done.record(main)
                pipe["free"][slot] = done
                if consume is not None:
                    with lock:
                        consume(e, sol)
                if k + 1 < len(energies):
                    ready = nxt if nxt is not None else self._generate(pipe, energies[k + 1], (k + 1) % nin)

    def run(self, energies, consume=None, timings=None):
        """Solve ``energies``; returns the number solved.  With several pipes,
        ``consume`` is called from the pipes' threads (serialised by a lock),
        in each pipe's energy order."""
        import threading

        energies = list(energies)
        if not energies:
            return 0
        self._caller = torch.cuda.current_stream(self.device)
        if self.overlap and self.concurrent == 1:
            return self._run_overlapped(energies, consume)
        lock = threading.Lock()
        k = min(self.concurrent, len(energies))
        shares = [energies[p::k] for p in range(k)]
        if k == 1:
            self._run_pipe(0, shares[0], consume, timings, lock)
        else:
            errors = []

            def work(p):
                try:
                    self._run_pipe(p, shares[p], consume, None, lock)
                except BaseException as exc:  # noqa: BLE001 - re-raised below
                    errors.append(exc)

            threads = [threading.Thread(target=work, args=(p,)) for p in range(k)]
            for t in threads:
                t.start()
            for t in threads:
                t.join()
            if errors:
                raise errors[0]
        for p in range(k):
            self._caller.wait_stream(self.pipes[p]["stream"])
        return len(energies)


    def _run_overlapped(self, energies, consume):
        """Energy k+1's forward sweeps (chain-bound: the Schur chains leave
        SMs idle) run while energy k's backward sweeps (tensor-pipe bound)
        do, on a second partition runner: two energies in flight with one
        output set.  Per energy: generate into input slot k % 2 (after the
        backward that read it), forward on runner k % 2, backward into the
        shared outputs (after the previous energy's outputs were consumed)."""
        from .dist import InGpuPartitions
        from .matrix import SelectedSolution

        dev = self.device
        if self._runners is None:
            shape = (self.n, self.b, self.a)
            self._runners = [InGpuPartitions(shape, self.mode, self.parts, dev, lane_base=p * self.parts, pipe=p)
                             for p in range(2)]
            self._pstreams = [torch.cuda.Stream(dev) for _ in range(2)]
        R, S = self._runners, self._pstreams
        pipe = self.pipes[0]
        for s_ in S:
            s_.wait_stream(self._caller)

        def forward(k, ready):
            with torch.cuda.device(dev), torch.cuda.stream(S[k % 2]):
                S[k % 2].wait_event(ready)
                A, B = pipe["inputs"][k % 2]
                return R[k % 2].run_forward(A, B)

        st = forward(0, self._generate(pipe, energies[0], 0))
        out_free = None
        for k, e in enumerate(energies):
            nxt = self._generate(pipe, energies[k + 1], (k + 1) % 2) if k + 1 < len(energies) else None
            with torch.cuda.device(dev), torch.cuda.stream(S[k % 2]):
                if out_free is not None:
                    S[k % 2].wait_event(out_free)
                R[k % 2].run_backward(st, out=self.out)
                done = torch.cuda.Event()
                done.record(S[k % 2])
            pipe["free"][k % 2] = done
            if nxt is not None:
                st = forward(k + 1, nxt)  # overlaps this backward on the GPU
            if consume is not None:
                done.synchronize()
                consume(e, SelectedSolution(x_a=self.out[0], x_b=self.out[1], mode=self.mode))
            out_free = done
        for s_ in S:
            self._caller.wait_stream(s_)
        return len(energies)


class HostEnergySweep:
    """Solve a sequence of energy points whose inputs and outputs live in
    pinned host memory, overlapping the PCIe traffic of neighbouring energies
    with the solves (the end-to-end form of config 4/5).

    Energy k: its inputs were copied host->device into input slot k % 2
    while energy k-1 solved (h2d stream); it solves into output slot
    ``k % out_slots``; its outputs are copied device->host on the d2h stream
    while energy k+1 solves.  PCIe is full duplex, so in steady state one
    energy costs max(solve, H2D, D2H) instead of the single-call
    max(forward, H2D) + max(backward, D2H).  Device memory: 2 input slots +
    ``out_slots`` output slots (cfg4: 16 GiB per matrix, 128 GiB at
    out_slots=2, plus the ~36 GiB solve workspace).  ``out_slots=1`` keeps one
    device output set and streams it out behind each backward sweep instead
    (``solve_selected``'s host-output path); ``None`` = 2 when the buffers
    fit.  With two slots the LAST energy streams its outputs out behind its
    backward into its slot (no whole-matrix drain after the final solve) and
    the first energy's inputs are loaded whole before it (streaming them
    behind its forward delayed the second energy's load; BSEL_SWEEP_STREAM_
    FIRST / _LAST switch both).  Config 4, 16 energies, round 2: 880 ms per
    energy (steady state ~818 ms per energy; device-resident 784 ms); round
    1: 1151 ms with 2 slots, 1200 ms with 1.  The two-slot form needs the
    solve's status / symmetry reads to bypass the copy engine (a small D2H
    waits behind the in-flight output D2H; they are published through mapped
    host memory, ``Context::publish_flags``).
    """

    def __init__(self, n: int, b: int, a: int, mode: str = "siq", device=None, partitions=None,
                 out_slots: int | None = None):
        if out_slots not in (None, 1, 2):
            raise ValueError("out_slots must be 1, 2 or None (2 when the buffers fit, else 1)")
        self.n, self.b, self.a, self.mode = n, b, a, mode
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.parts = default_partitions(n) if partitions is None else partitions
        fused = mode == "siq"
        mk = lambda: DeviceBta.empty(n, b, a, self.device, zero=False)  # noqa: E731
        self.inputs = [(mk(), mk() if fused else None) for _ in range(2)]
        self.out = None
        if out_slots != 1:
            try:
                self.out = [(mk(), mk() if fused else None) for _ in range(2)]
            except torch.cuda.OutOfMemoryError:
                if out_slots == 2:
                    raise
                torch.cuda.empty_cache()
        self.out_slots = 2 if self.out is not None else 1
        self._auto_slots = out_slots is None
        self.h2d = torch.cuda.Stream(self.device)
        self.d2h = torch.cuda.Stream(self.device)

    @staticmethod
    def _chunked(host_m, dev_m, to_host):
        """Whole-matrix copy as ~32 MiB pieces: a multi-GiB copy holds its
        copy engine for hundreds of ms, and the solve's own small copies
        queued behind it would stall the sweeps."""
        for k, arr in host_m.stacked().items():
            if not arr.size:
                continue
            h, d = torch.from_numpy(arr), getattr(dev_m, k)
            step = max(1, (32 << 20) // max(1, arr[0].nbytes)) if arr.ndim == 3 else len(arr)
            for i in range(0, len(arr), step):
                if to_host:
                    h[i:i + step].copy_(d[i:i + step], non_blocking=True)
                else:
                    d[i:i + step].copy_(h[i:i + step], non_blocking=True)

    def _load(self, host, slot, free):
        a, b = host
        A, B = self.inputs[slot]
        with torch.cuda.device(self.device), torch.cuda.stream(self.h2d):
            if free is not None:
                self.h2d.wait_event(free)
            self._chunked(a, A, False)
            if B is not None:
                self._chunked(b, B, False)
            ready = torch.cuda.Event()
            ready.record(self.h2d)
        return ready

    def run(self, inputs, outputs, timings=None):
        """Solve energies ``inputs[k] = (a_k, b_k)`` (pinned host BtaMatrix)
        into ``outputs[k] = (x_a_k, x_b_k)`` (pinned host BtaMatrix); returns
        once every output is on the host."""
        inputs, outputs = list(inputs), list(outputs)
        if len(inputs) != len(outputs):
            raise ValueError("inputs and outputs differ in length")
        if not inputs:
            return 0
        main = torch.cuda.current_stream(self.device)
        self.h2d.wait_stream(main)  # the first load is ordered after the caller's queued work
        in_free = [None, None]  # event: solve no longer reads the input slot
        out_free = [None, None]  # event: D2H of the output slot finished
        # The partitioned solve streams host inputs in behind its forward
        # sweeps: the first energy uses that (no unoverlapped fill), and the
        # second energy's load starts once the first's inputs are in.  (Round
        # 1 measured 8.5 s for a streamed first energy with device outputs:
        # solve_selected copied the caller's device outputs to pageable host
        # memory for host inputs -- fixed in rgf.py.)
        # Streaming the first energy's inputs behind its forward finishes it
        # sooner but delays the second (its load then starts only after those
        # inputs): config 4, 16 energies, 908 vs 898 ms per energy with the
        # plain first load (tools/e2e_probe.py) -- off by default.
        stream_first = (self.parts > 1 and self.n >= 2 * self.parts
                        and os.environ.get("BSEL_SWEEP_STREAM_FIRST", "0") != "0")
        self._stream_last = os.environ.get("BSEL_SWEEP_STREAM_LAST", "1") != "0"
        self.done_events = []
        ready = None if stream_first else self._load(inputs[0], 0, None)
        k = 0
        preloaded = None  # next energy's load already enqueued (OOM retry)
        while k < len(inputs):
            host_in, host_out = inputs[k], outputs[k]
            s = k & 1
            first = stream_first and k == 0
            nxt = None
            if k + 1 < len(inputs) and not first:
                nxt = preloaded if preloaded is not None else self._load(inputs[k + 1], s ^ 1, in_free[s ^ 1])
            preloaded = None
            if ready is not None:
                main.wait_event(ready)
            A, B = self.inputs[s]
            src = host_in if first else (A, B)
            kw = {}
            if first:
                # the host-output solve synchronizes before it returns: the
                # next energy's load is enqueued from the callback, right after
                # this energy's last streamed input chunk (not after its solve)
                held = []
                io = {}
                if k + 1 < len(inputs):
                    io["on_inputs_done"] = lambda ev: held.append(self._load(inputs[k + 1], s ^ 1, ev))
                kw = {"_device_in": (A, B), "_io_events": io}
            # The last energy streams its outputs out behind its backward sweeps
            # (the form out_slots=1 uses for every energy): a whole-matrix D2H
            # after its solve would be an unoverlapped 34 GB drain at config 4.
            last_streamed = self.out is not None and k == len(inputs) - 1 and k > 0 and self._stream_last
            if self.out is None or last_streamed:
                if last_streamed:  # device storage behind the streamed outputs: this energy's output slot
                    if out_free[k % 2] is not None:
                        main.wait_event(out_free[k % 2])
                    kw["_device_out"] = self.out[k % 2]
                solve_selected(src[0], src[1], self.mode, out=host_out, partitions=self.parts, timings=timings,
                               **kw)
                done = torch.cuda.Event(enable_timing=True)
                done.record(main)
            else:
                o = k % self.out_slots
                if out_free[o] is not None:
                    main.wait_event(out_free[o])
                XA, XB = self.out[o]
                try:
                    solve_selected(src[0], src[1], self.mode, out=(XA, XB), partitions=self.parts,
                                   timings=timings, **kw)
                except torch.cuda.OutOfMemoryError:
                    # The solve workspace is allocated lazily by the first
                    # solve: when two output slots leave too little room for
                    # it, fall back to one slot (outputs streamed behind the
                    # backward) and redo this energy.  Nothing of it has
                    # reached the host yet.
                    if not self._auto_slots or k != 0:
                        raise
                    self.out = None
                    self.out_slots = 1
                    torch.cuda.empty_cache()
                    preloaded = nxt
                    continue
                done = torch.cuda.Event(enable_timing=True)
                done.record(main)
                with torch.cuda.device(self.device), torch.cuda.stream(self.d2h):
                    self.d2h.wait_event(done)
                    self._chunked(host_out[0], XA, True)
                    if XB is not None:
                        self._chunked(host_out[1], XB, True)
                    ev = torch.cuda.Event()
                    ev.record(self.d2h)
                    out_free[o] = ev
            in_free[s] = done
            self.done_events.append(done)
            if first and held:
                nxt = held[0]
            ready = nxt
            k += 1
        main.wait_stream(self.d2h)
        main.wait_stream(self.h2d)
        main.synchronize()
        return len(inputs)
