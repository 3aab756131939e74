#!/usr/bin/env python
"""Benchmark: ms per energy point of the fused BTA SI+SQ solve (BASELINE.json).

Workload at N=1: BASELINE config 4 (the north-star shape, fits one B200):
BTA n_blocks=1024, block=512, tip=256, complex128, bench-protocol synthetic
inputs A = generate_dd_bta(seed 0), B = hermitianize(generate_dd_bta(seed 1))
generated on the device (same splitmix64 stream as the reference generator).
A "step" = one full SI+SQ solve of one energy point.  N>1 (torchrun): the
same energy point partitioned across N GPUs with the paper's distributed
scheme (strong scaling).

Prints ONE JSON line (rank 0).  `value` is device-timed with inputs resident
in HBM (inputs = 32 GiB >> 126 MB L2, so no flush is needed); `e2e` is the
same metric through the public API with pinned host buffers (H2D of A, B and
D2H of X_A, X_B inside the timed region).  `--impl reference` times the CPU
reference path (the oracle port of btasel on the host cores) on a bounded
sample and extrapolates to the full workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# NCCL's version banner goes to stdout, which must carry only the JSON line.
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"
sys.path.insert(0, ROOT)
# stdout carries only the JSON line: everything else written to fd 1 (NCCL
# banners, library prints) is redirected to stderr; emit() writes the line
# to the saved original stdout.
_JSON_FD = os.dup(1)
os.dup2(2, 1)


def emit(line):
    os.write(_JSON_FD, (json.dumps(line) + "\n").encode())

WORKLOADS = {
    # name: (n, b, a, config index in BASELINE.json)
    "cfg4": (1024, 512, 256, 3),
    "cfg3": (128, 512, 64, 2),
    "cfg2": (64, 256, 0, 1),
    "cfg5": (256, 1024, 256, 4),
}
FP64_PEAK_FILE = os.path.join(ROOT, "profiles", "fp64_peak_r01.json")
NCU_TRAFFIC_FILE = os.path.join(ROOT, "profiles", "ncu_gemm3m_step_r02.json")
METRIC = "ms per energy point, fused BTA SI+SQ at 1/2/4/8 B200; % FP64 TC peak"


def gemm_rate_by_phase(path, keep=False):
    """The GEMM kernel's executed rate per phase from the per-launch timeline
    of the profiled step (BSEL_PROFILE_DUMP: kind, stream, start, end,
    algorithmic flops, executed flops): forward = until the last block
    inverse ends, backward = after.  Rate = executed flops of the phase's
    GEMM launches / union of their spans."""
    try:
        rows = []
        with open(path) as fh:
            for line in fh:
                p = line.strip().split(",")
                if len(p) >= 6:
                    rows.append((int(p[0]), float(p[2]), float(p[3]), float(p[4]), float(p[5])))
        if not keep:
            os.remove(path)
    except OSError:
        return None
    if not rows:
        return None
    inv_end = max((r[2] for r in rows if r[0] == 1), default=None)
    if inv_end is None:
        return None
    out = {}
    for name, sel in (("forward", lambda r: r[2] <= inv_end), ("backward", lambda r: r[1] >= inv_end)):
        g = sorted((r for r in rows if r[0] == 0 and sel(r)), key=lambda r: r[1])
        busy, c0, c1 = 0.0, None, None
        for r in g:
            if c1 is None or r[1] > c1:
                if c1 is not None:
                    busy += c1 - c0
                c0, c1 = r[1], r[2]
            else:
                c1 = max(c1, r[2])
        if c1 is not None:
            busy += c1 - c0
        ex = sum(r[4] for r in g)
        out[name] = {"gemm_busy_ms": round(busy, 2), "gemm_executed_tflops": ex / (busy * 1e-3) / 1e12 if busy else None,
                     "gemm_launches": len(g)}
    return out


def flops_seq(n, b, a, mode="siq"):
    """Reference sequential op inventory (8 real flops per complex MAC, 8N^3
    per inverse), summed from the per-step tables (kernels.record_sweep)."""
    from paper_2601_04904_b200.kernels import OpCounter, record_sweep

    c = OpCounter(b=b, a=a)
    record_sweep(c, n, b, a, mode, "forward")
    record_sweep(c, n, b, a, mode, "backward")
    dim = {"b": b, "a": a}
    total = 0.0
    for label, cnt in c.gemm_by_shape.items():
        m, k, nn = (dim[ch] if ch in dim else 0 for ch in label)
        total += 8.0 * m * k * nn * cnt
    total += 8.0 * n * b ** 3 + (8.0 * a ** 3 if a else 0.0)
    return total


def fp64_peak_tflops():
    try:
        with open(FP64_PEAK_FILE) as fh:
            d = json.load(fh)
        return max(d["dmma_m8n8k4_w8_tflops"], d["dmma_m8n8k4_w16_tflops"]), "measured DMMA mma.sync f64 loop (profiles/fp64_peak_r01.json)"
    except Exception:  # pragma: no cover
        return 37.2, "nominal 148 SM x 128 flop/clk x 1965 MHz"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.dev)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._pump, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[4:8]):
                if flag.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if mx and s > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_impl():
    """(module, kind): the unmodified reference btasel installed in
    baseline/_ref (pip install --target) -> "reference";
    otherwise the oracle port (oracle/, same NumPy/SciPy arithmetic) ->
    "port"."""
    if os.path.isdir(os.path.join(REF_DIR, "btasel")):
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        try:
            import btasel

            return btasel, "reference"
        except Exception:  # pragma: no cover - broken install
            pass
    import oracle  # CPU baseline leg only

    return oracle, "port"


def set_host_blas_threads(count):
    """All host cores for the CPU reference path.  torchrun exports
    OMP_NUM_THREADS=1 to every rank, which would make OpenBLAS single-threaded:
    use the reference's own pool control (btasel.set_blas_threads,
    threads.py:41-70), else threadpoolctl."""
    ref, _ = reference_impl()
    if hasattr(ref, "set_blas_threads"):
        ref.set_blas_threads(count)
        return
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(count)
    except Exception:  # pragma: no cover
        pass


def cpu_sample(n_s, b, a, threads=None):
    """Time the CPU reference path (btasel solve_selected, or its oracle port,
    NumPy/SciPy on the host BLAS) on an n_s-block sample of the workload with
    the reference bench protocol inputs (bench.py:202-203).  Returns seconds."""
    ref, _ = reference_impl()
    set_host_blas_threads(threads or host_cores())
    A = ref.generate_dd_bta(n_s, b, a, seed=0)
    B = ref.hermitianize(ref.generate_dd_bta(n_s, b, a, seed=1))
    t0 = time.perf_counter()
    ref.solve_selected(A, B, "siq")
    return time.perf_counter() - t0


def host_info():
    """CPU model, RAM and BLAS of the host the CPU reference runs on."""
    info = {"nproc": os.cpu_count(), "cores_used": host_cores()}
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    info["cpu_model"] = line.split(":", 1)[1].strip()
                    break
        with open("/proc/meminfo") as fh:
            info["ram_gib"] = round(int(fh.readline().split()[1]) / 2**20, 1)
    except OSError:
        pass
    try:
        from threadpoolctl import threadpool_info

        blas = [x for x in threadpool_info() if x.get("user_api") == "blas"]
        if blas:
            info["blas"] = f"{blas[0].get('internal_api')} {blas[0].get('version')}"
    except Exception:
        pass
    return info


def cpu_baseline_protocol(n, b, a, n_all=8, n_one=2, repeats=3):
    """The CPU reference path timed as BASELINE.md 4 asks, bounded to ~30 s:
    the unmodified reference (or its port) on n_all blocks with BLAS threads
    = all host cores (median of `repeats`) and on n_one blocks with 1 thread,
    each extrapolated linearly in n (acceptance criterion 7); the faster is
    the baseline.  The unbounded protocol (n in {32, 64, 128}, linear fit,
    both thread counts) is tools/cpu_protocol.py -> profiles/."""
    t_all = statistics.median(cpu_sample(n_all, b, a) for _ in range(repeats))
    t_one = cpu_sample(n_one, b, a, threads=1)
    ms_all, ms_one = t_all / n_all * n * 1e3, t_one / n_one * n * 1e3
    return {"all_cores_ms": ms_all, "one_thread_ms": ms_one, "value": min(ms_all, ms_one),
            "t_all_s": t_all, "t_one_s": t_one, "n_all": n_all, "n_one": n_one, "repeats": repeats}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, n, b, a):
    """--impl reference: CPU reference path on rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_s = args.cpu_sample_n
    for _ in range(args.warmup):
        cpu_sample(n_s, b, a)
    times = [cpu_sample(n_s, b, a) for _ in range(args.steps)]
    per = statistics.mean(times) / n_s * n * 1e3
    _, kind = reference_impl()
    what = ("unmodified reference btasel (baseline/_ref)" if kind == "reference" else "oracle port of btasel")
    sample = (f"{what} solve_selected (NumPy/SciPy, OpenBLAS on all {host_cores()} host cores) on "
              f"n={n_s} of {n} blocks (b={b}, a={a}), extrapolated linearly in n (reference acceptance "
              f"criterion 7)")
    cores = host_cores()
    line = {
        "impl": "reference", "metric": METRIC, "value": per, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": args.workload, "n_blocks": n, "block": b, "tip": a, "mode": "siq"},
        "cpu_baseline": {"value": per, "unit": "ms", "cores": cores, "kind": kind, "sample": sample,
                         "host": host_info(), "step_s": [round(t, 3) for t in times]},
        "e2e": {"value": per, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def pipelined_e2e(args, n, b, a, parts, hA, hB, hXA, hXB, single):
    """End to end through ``HostEnergySweep``: K energy points, each one's
    inputs copied host->device and outputs device->host inside the timed
    region, the copies of neighbouring energies overlapped with the solves
    (every step moves the same bytes as the single-call form; the same
    pinned host buffers serve every energy)."""
    import gc

    import torch

    import paper_2601_04904_b200 as bs

    gc.collect()
    torch.cuda.empty_cache()
    free_gib = torch.cuda.mem_get_info()[0] / 2**30
    # out_slots: 2 when the double-buffered outputs fit (BSEL_E2E_OUT_SLOTS forces 1 or 2)
    want = int(os.environ["BSEL_E2E_OUT_SLOTS"]) if os.environ.get("BSEL_E2E_OUT_SLOTS") else None
    try:
        sweep = bs.HostEnergySweep(n, b, a, "siq", partitions=parts, out_slots=want)
    except torch.cuda.OutOfMemoryError:
        return dict(single, pipelined_note="HostEnergySweep buffers do not fit")
    slots = sweep.out_slots
    k = max(args.steps, args.e2e_energies)
    sweep.run([(hA, hB)] * 2, [(hXA, hXB)] * 2)  # warm (both slots)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    sweep.run([(hA, hB)] * k, [(hXA, hXB)] * k)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / k
    del sweep
    gc.collect()
    torch.cuda.empty_cache()
    return {"value": ms, "unit": "ms", "h2d_bytes_per_step": single["h2d_bytes_per_step"],
            "d2h_bytes_per_step": single["d2h_bytes_per_step"],
            "api": f"HostEnergySweep.run: {k} energy points from/to pinned host buffers, H2D of energy k+1 "
                   f"and D2H of energy k-1 overlapped with energy k's solve (out_slots={slots}; the last "
                   "energy's outputs stream out behind its backward); timed region includes the first H2D "
                   "and the last D2H",
            "single_call_ms": single["value"], "single_call_api": single["api"],
            "device_free_gib_before": round(free_gib, 1)}


def dist_e2e(args, solver, A, B, n, world, rank, dev, dist):
    """N>1 end-to-end through DistSolver.solve(host_in, host_out): every step
    each rank streams the input blocks it needs from pinned host memory
    (its partition chunk by chunk behind its forward sweep, plus the other
    partitions' separators and the tip) and streams the solution blocks it
    owns back behind its backward sweep (outputs stay sharded).  Host
    storage per rank = HostWindow (only the blocks that rank touches)."""
    import torch
    import paper_2601_04904_b200 as bs

    lo, hi = solver.owned_range()
    seps = [solver.plan.ranges[p][1] - 1 for p in range(solver.plan.num_parts - 1)]
    hin = tuple(bs.HostWindow(n, A.b, A.a, lo, hi, seps).fill_from(M) for M in (A, B))
    hout = tuple(bs.HostWindow(n, A.b, A.a, lo, hi) for _ in (A, B))
    torch.cuda.synchronize()
    solver.solve(host_in=hin, host_out=hout)
    torch.cuda.synchronize()
    # One streamed call per energy (default), or BSEL_DIST_E2E=pipelined:
    # DistSolver.solve_energies (energy k+1's window copied in and energy
    # k-1's outputs copied out while energy k solves) when its extra device
    # input / output sets fit on every rank.  At 2 GPUs the pipelined form
    # measured 882 vs 822 ms: the ranks share the host's PCIe / memory
    # bandwidth (68.6 GB per energy in total), which bounds both forms.
    form = "single"
    if os.environ.get("BSEL_DIST_E2E", "single") == "pipelined" and solver.k == 1:
        try:
            solver.solve_energies([hin] * 2, [hout] * 2)  # warm: allocates the second slots
            torch.cuda.synchronize()
            form = "pipelined"
        except torch.cuda.OutOfMemoryError:
            solver._slot1 = None
            torch.cuda.empty_cache()
    ok = torch.tensor([1.0 if form == "pipelined" else 0.0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    form = "pipelined" if ok.item() > 0 else "single"
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    if form == "pipelined":
        solver.solve_energies([hin] * args.steps, [hout] * args.steps)
    else:
        for _ in range(args.steps):
            solver.solve(host_in=hin, host_out=hout)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    # bytes actually moved per step: inputs of the window (tip once per rank),
    # outputs = the blocks this rank owns (+ the tip on rank 0)
    h2d = sum(w.nbytes for w in hin)
    d2h = sum(w.nbytes - w.tip.numel() * 16 * (rank != 0) for w in hout)
    stats = torch.tensor([ms, h2d, d2h], dtype=torch.float64, device=dev)
    mx = stats[:1].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    dist.all_reduce(stats, op=dist.ReduceOp.SUM)
    return {"value": float(mx.item()), "unit": "ms", "h2d_bytes_per_step": int(stats[1].item()),
            "d2h_bytes_per_step": int(stats[2].item()),
            "form": form,
            "note": ("per rank: its partition + separators + tip copied host->device for energy k+1 and its "
                     "owned solution blocks of energy k-1 copied back while energy k solves "
                     "(DistSolver.solve_energies, steps = energies, first load and last copy-out timed)"
                     if form == "pipelined" else
                     "per rank: its partition + separators + tip streamed in behind the forward, its owned "
                     "solution blocks streamed out behind the backward; max over ranks")}


def cfg5_side_measurement(args, dev):
    """BASELINE configs[4] (energy sweep, n=256, b=1024, a=256) at N=1 as a
    side key of the default line: the cfg4 buffers are released first, then
    2 warm-up + args.cfg5_energies timed energies through EnergySweep
    (overlapped energies when they fit), device-timed ms per energy."""
    import gc

    import torch

    import paper_2601_04904_b200 as bs

    try:
        bs.release_caches()
        gc.collect()
        torch.cuda.empty_cache()
        n, b, a, idx = WORKLOADS["cfg5"]
        sweep = bs.EnergySweep(n, b, a, "siq", device=dev)
        sweep.run([0, 1])  # warm-up: 2 energies (the first batch after the cfg4 run is ~5 % slower)
        torch.cuda.synchronize()
        k = max(2, args.cfg5_energies)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        sweep.run(list(range(2, k + 2)))
        e.record()
        torch.cuda.synchronize()
        out = {"workload": f"cfg5: BASELINE.json configs[{idx}]", "n_blocks": n, "block": b, "tip": a,
               "ms_per_energy": s.elapsed_time(e) / k, "energies": k,
               "mode": "energy k+1's forward overlapped with energy k's backward" if sweep.overlap
               else "energies back to back",
               "note": "energies e = generator seeds (2e, 2e+1), generated on the device; device-timed"}
        del sweep
        gc.collect()
        torch.cuda.empty_cache()
        return out
    except Exception as exc:  # noqa: BLE001 - a side key must not lose the main line
        return {"error": f"{type(exc).__name__}: {exc}"}


def run_energy_sweep(args, n, b, a, cfg_idx, world, rank, local, dev, dist):
    """Config 5: energy-point sweep, energy parallel across ranks (weak
    scaling: ``--energies-per-gpu`` energies per GPU per step, no
    collective).  A step = every rank solves its energies; value = the
    step's device time (max over ranks) / all energies of the step."""
    import torch

    import paper_2601_04904_b200 as bs

    E = args.energies_per_gpu
    sweep = bs.EnergySweep(n, b, a, "siq", device=dev, concurrent=args.energy_concurrent or 1,
                           overlap=False if args.no_energy_overlap else None)
    mine = list(range(rank * E, (rank + 1) * E))  # energies of this rank (round robin over 64 = same set)

    def step():
        sweep.run(mine)

    t0 = time.perf_counter()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    warm_s = time.perf_counter() - t0
    launches0 = bs.kernel_launches()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        start.record()
        marks = []
        for _ in range(args.steps):
            step()
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append(ev)
        end.record()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms = start.elapsed_time(end) / args.steps
    step_ms = [round(start.elapsed_time(marks[0]), 1)] + [round(marks[i - 1].elapsed_time(marks[i]), 1)
                                                          for i in range(1, len(marks))]
    launches = (bs.kernel_launches() - launches0) // args.steps
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # executed flops of one energy point (GEMM products + inverses)
    from paper_2601_04904_b200 import _native

    prof = _native.Profile()
    lib = _native.load_library()
    lib.bsel_profile_begin()
    sweep.run(mine[:1])
    lib.bsel_profile_end(prof)
    if rank == 0:
        total_e = E * world
        per = ms / total_e
        F = flops_seq(n, b, a)
        Fx = prof.gemm_flops + prof.inverse_flops
        peak, peak_src = fp64_peak_tflops()
        tf = Fx * total_e / (ms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": per, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (device splitmix64 generator; energy e = seeds (2e, 2e+1))",
            "config": {"workload": f"cfg5: BASELINE.json configs[{cfg_idx}]", "n_blocks": n, "block": b, "tip": a,
                       "mode": "siq", "energies_per_gpu": E, "energies_per_step": total_e,
                       "parallelism": f"energy parallel over {world} GPU(s), 2 in-GPU partitions per energy, "
                                      + ("energy k+1's forward overlapped with energy k's backward" if sweep.overlap
                                         else f"{sweep.concurrent} energy pipe(s) per GPU"),
                       "l2": "inputs 28 GiB per energy >> L2"},
            "fp64_tflops_step": tf, "pct_fp64_peak_step": 100.0 * tf / (peak * world), "flops_per_energy": Fx,
            "flops_reference_inventory_per_energy": F,
            "effective_tflops_reference_inventory": F * total_e / (ms * 1e-3) / 1e12,
            "roofline": {"bound": "tensor", "kernel": "whole step (DMMA GEMMs + inverses)",
                         "achieved": tf / world, "peak": peak, "unit": "TFLOP/s", "frac": tf / world / peak,
                         "traffic": None, "peak_source": peak_src},
            "gpu_launches": launches, "clocks": clk.summary(),
            "e2e": None, "e2e_note": "cfg5 inputs are generated on the device per energy (28 GiB each); "
                                    "host-resident energy sets are out of scope of this mode",
            "cpu_baseline": None, "warmup_s": warm_s,
        }
        emit(line)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS))
    ap.add_argument("--n", type=int, default=None, help="override n_blocks (debug)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-pipelined-e2e", action="store_true",
                    help="report the single-call e2e only (skip the HostEnergySweep measurement)")
    ap.add_argument("--e2e-energies", type=int, default=16,
                    help="energy points in the pipelined e2e run (max with --steps); the unoverlapped "
                         "first H2D and last D2H are amortised over them")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample-n", type=int, default=8)
    ap.add_argument("--partitions", type=int, default=None,
                    help="N=1: in-GPU partitions of solve_selected (default: library default)")
    ap.add_argument("--no-seq", action="store_true", help="skip the extra sequential-RGF measurement")
    ap.add_argument("--parts-per-gpu", type=int, default=int(os.environ.get("BSEL_PARTS_PER_GPU", "1")),
                    help="N>1: partitions per GPU (lanes), plan over N x this many partitions")
    ap.add_argument("--no-other-b", action="store_true",
                    help="skip the general / anti-Hermitian right-hand-side timings")
    ap.add_argument("--no-cfg5", action="store_true", help="N=1: skip the config-5 side measurement")
    ap.add_argument("--cfg5-energies", type=int, default=8, help="N=1: timed energies of the config-5 side key")
    ap.add_argument("--energy-concurrent", type=int, default=None,
                    help="cfg5: independent energy pipes per GPU (default 1)")
    ap.add_argument("--no-energy-overlap", action="store_true",
                    help="cfg5: no overlap of energy k+1's forward with energy k's backward")
    ap.add_argument("--energies-per-gpu", type=int, default=8,
                    help="cfg5: energy points per GPU per step (64 energies on 8 GPUs)")
    args = ap.parse_args()
    n, b, a, cfg_idx = WORKLOADS[args.workload]
    if args.n:
        n = args.n
    if args.impl == "reference":
        return run_reference(args, n, b, a)

    import torch

    import paper_2601_04904_b200 as bs
    from paper_2601_04904_b200 import _native

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # pinned host buffers (e2e) on this GPU's NUMA node; the CPU-baseline leg
    # restores the full affinity
    all_cpus = bs.bind_host_to_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)
        from paper_2601_04904_b200 import dist as bdist

    if args.workload == "cfg5":
        return run_energy_sweep(args, n, b, a, cfg_idx, world, rank, local, dev, dist)

    # ---- inputs, generated on device --------------------------------------
    t_gen = time.perf_counter()
    A = bs.generate_dd_bta_device(n, b, a, seed=0, device=dev)
    B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1, device=dev))
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen

    parts = 1
    if world == 1:
        XA, XB = bs.DeviceBta.empty(n, b, a, dev, zero=False), bs.DeviceBta.empty(n, b, a, dev, zero=False)
        ctx = _native.Context.get(local)
        ws = torch.empty(ctx.workspace_bytes(n, b, a, True), dtype=torch.uint8, device=dev)

        parts = args.partitions if args.partitions else bs.default_partitions(n)

        def step():
            bs.solve_selected(A, B, "siq", out=(XA, XB), workspace=ws, partitions=parts)
    else:
        # Partition sizes from per-block costs measured on B200 (end : middle
        # = 1 : 2.05 -> [344, 168, 168, 344] at 4 GPUs: 321-323 vs 331 ms with
        # the reference's product-count plan [354, 158, 158, 354], whose
        # middles waited ~30 ms at the exchange; profiles/sweeps_r02.md).
        # Results agree with the reference plan's to rounding (the parity
        # tests and dist_solve use the reference plan).  BSEL_PLAN_COSTS=
        # "end,mid" overrides, "ref" restores the reference's plan.
        pc = os.environ.get("BSEL_PLAN_COSTS", "1,2.05")
        plan_costs = None if pc in ("", "ref") else tuple(float(x) for x in pc.split(","))
        solver = bdist.DistSolver(A, B, "siq", world, rank, dev, plan_costs=plan_costs,
                                  parts_per_rank=args.parts_per_gpu)

        def step():
            solver.solve()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- device-resident timed region --------------------------------------
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = bs.kernel_launches()
    with ClockSampler(local) as clk:
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        start.record()
        marks = []
        for _ in range(args.steps):
            step()
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            marks.append(ev)
        end.record()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
    ms = start.elapsed_time(end) / args.steps
    step_ms = [round(start.elapsed_time(marks[0]), 1)] + [round(marks[i - 1].elapsed_time(marks[i]), 1)
                                                          for i in range(1, len(marks))]
    launches = (bs.kernel_launches() - launches0) // args.steps
    if dist:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = clk.summary()

    phases = {}
    seq_ms = None
    if world == 1:
        bs.solve_selected(A, B, "siq", out=(XA, XB), workspace=ws, timings=phases, partitions=parts)
        if parts > 1 and not args.no_seq:
            # the pure sequential RGF sweeps (rgf.py order), for reference
            bs.solve_selected(A, B, "siq", out=(XA, XB), workspace=ws, partitions=1)
            s1, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s1.record()
            for _ in range(2):
                bs.solve_selected(A, B, "siq", out=(XA, XB), workspace=ws, partitions=1)
            e1.record()
            torch.cuda.synchronize()
            seq_ms = s1.elapsed_time(e1) / 2
    else:
        phases = solver.phase_seconds()
    phases = {k: v * 1e3 for k, v in phases.items()}
    rank_phases = None
    if dist:
        keys = sorted(phases)
        t = torch.tensor([phases[k] for k in keys], device=dev, dtype=torch.float64)
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        rank_phases = [{k: round(float(v), 2) for k, v in zip(keys, x.tolist())} for x in allt]

    # ---- live per-kernel timing of the dominant kernel (one extra step) ----
    # Every launch is bracketed by CUDA events on its own stream; launches of
    # the concurrent streams overlap, so the kernel's time is the UNION of its
    # launch spans (busy time) and its rate = its algorithmic flops / busy time.
    prof = _native.Profile()
    lib = _native.load_library()
    import tempfile

    dump = os.path.join(tempfile.gettempdir(), f"bsel_timeline_{os.getpid()}.csv")
    os.environ.setdefault("BSEL_PROFILE_DUMP", dump)  # read by the library at its first profile_end
    lib.bsel_profile_begin()
    pstart, pend = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pstart.record()
    step()
    pend.record()
    lib.bsel_profile_end(prof)
    prof_ms = pstart.elapsed_time(pend)
    by_phase = gemm_rate_by_phase(os.environ["BSEL_PROFILE_DUMP"], keep=os.environ["BSEL_PROFILE_DUMP"] != dump)
    peak, peak_src = fp64_peak_tflops()
    ncu = None
    if os.path.exists(NCU_TRAFFIC_FILE):
        with open(NCU_TRAFFIC_FILE) as f:
            ncu = json.load(f)
    # the GEMM kernel's rate over its busy time: EXECUTED tensor-pipe flops
    # (3M kernel: 6 M N K per complex product, real-embedding kernel: 8 M N K)
    # and ALGORITHMIC flops (8 M N K, the reference's counting)
    busy_s = prof.gemm_busy_ms * 1e-3
    gemm_tflops = prof.gemm_exec_flops / busy_s / 1e12 if busy_s > 0 else None
    gemm_tflops_alg = prof.gemm_flops / busy_s / 1e12 if busy_s > 0 else None
    # executed flops of one step (all ranks): GEMM products + block inverses
    executed = prof.gemm_exec_flops + prof.inverse_flops
    algorithmic = prof.gemm_flops + prof.inverse_flops
    if dist:
        t = torch.tensor([executed, algorithmic], device=dev, dtype=torch.float64)
        dist.all_reduce(t)
        executed, algorithmic = (float(x) for x in t.tolist())
    F = flops_seq(n, b, a)
    achieved_step = executed / (ms * 1e-3) / 1e12

    # ---- other right-hand sides (N=1): general B and anti-Hermitian B -----
    other_b = {}
    if world == 1 and not args.no_other_b:
        Bg = bs.generate_dd_bta_device(n, b, a, seed=1, device=dev)  # general (not hermitianized)
        for name, Bx in (("general", Bg), ("antihermitian", None)):
            if Bx is None:  # i * hermitianize(B): B = -B^H exactly (lesser/greater self-energies)
                Bx = Bg
                bs.hermitianize_device(Bx)
                for t_ in Bx.tensors().values():
                    t_.mul_(1j)
            bs.solve_selected(A, Bx, "siq", out=(XA, XB), workspace=ws, partitions=parts)
            torch.cuda.synchronize()
            s3, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s3.record()
            for _ in range(2):
                bs.solve_selected(A, Bx, "siq", out=(XA, XB), workspace=ws, partitions=parts)
            e3.record()
            torch.cuda.synchronize()
            other_b[name] = s3.elapsed_time(e3) / 2
        del Bg, Bx
        torch.cuda.empty_cache()

    # ---- end-to-end through the public API with pinned host buffers -------
    e2e = None
    if not args.no_e2e and world == 1:
        hA = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
        hB = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
        A.copy_to_host(hA)
        B.copy_to_host(hB)
        del XA, XB
        A = B = None
        torch.cuda.empty_cache()
        hXA = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
        hXB = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
        bs.solve_selected(hA, hB, "siq", out=(hXA, hXB), workspace=ws, partitions=parts)  # warm allocator
        torch.cuda.synchronize()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        for _ in range(args.steps):
            bs.solve_selected(hA, hB, "siq", out=(hXA, hXB), workspace=ws, partitions=parts)
        e2.record()
        torch.cuda.synchronize()
        e2e_ms = s2.elapsed_time(e2) / args.steps
        e2e = {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": hA.nbytes + hB.nbytes,
               "d2h_bytes_per_step": hXA.nbytes + hXB.nbytes,
               "api": "solve_selected(host pinned A, B, out=host pinned X_A, X_B), one call per step"}
        if not args.no_pipelined_e2e:
            ws = None  # the sequential-path workspace is not used by the partitioned sweep
            e2e = pipelined_e2e(args, n, b, a, parts, hA, hB, hXA, hXB, e2e)
    elif not args.no_e2e:
        e2e = dist_e2e(args, solver, A, B, n, world, rank, dev, dist)

    # ---- CPU baseline (rank 0, N=1 only) -----------------------------------
    cpu = None
    if not args.no_cpu and world == 1 and rank == 0:
        if all_cpus:
            os.sched_setaffinity(0, all_cpus)
        pr = cpu_baseline_protocol(n, b, a, n_all=args.cpu_sample_n)
        _, kind = reference_impl()
        what = "reference btasel (baseline/_ref)" if kind == "reference" else "oracle port"
        faster_all = pr["all_cores_ms"] <= pr["one_thread_ms"]
        cpu = {"value": pr["value"], "unit": "ms", "cores": host_cores() if faster_all else 1, "kind": kind,
               "sample": f"{what} solve_selected (NumPy/SciPy/OpenBLAS), bench-protocol inputs: n={pr['n_all']} of "
                         f"{n} blocks (b={b}, a={a}) with BLAS threads = all {host_cores()} cores, median of "
                         f"{pr['repeats']} ({pr['t_all_s']:.2f} s), and n={pr['n_one']} with 1 thread "
                         f"({pr['t_one_s']:.2f} s); each extrapolated linearly in n (acceptance criterion 7); "
                         f"value = the faster",
               "all_cores_ms": pr["all_cores_ms"], "one_thread_ms": pr["one_thread_ms"], "host": host_info()}
        full = os.path.join(ROOT, "profiles", "cpu_protocol_r02.json")
        try:
            with open(full) as fh:
                cpu["full_protocol"] = {k: v for k, v in json.load(fh).items() if k in ("value_ms", "fit", "host")}
            cpu["full_protocol"]["source"] = "profiles/cpu_protocol_r02.json (tools/cpu_protocol.py on this pool)"
        except (OSError, ValueError):
            pass

    # ---- config 5 side measurement (N=1): the energy sweep's ms per energy -
    cfg5 = None
    if world == 1 and not args.no_cfg5:
        A = B = XA = XB = ws = None  # noqa: F841 - release the cfg4 device buffers first
        hA = hB = hXA = hXB = None  # noqa: F841 - and the 69 GB of pinned host buffers of the e2e leg
        cfg5 = cfg5_side_measurement(args, dev)

    if rank == 0:
        line = {
            "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (device splitmix64 generator, bench protocol seeds 0/1)",
            "config": {"workload": f"{args.workload}: BASELINE.json configs[{cfg_idx}]", "n_blocks": n, "block": b,
                       "tip": a, "mode": "siq",
                       "parallelism": (f"partitions{world * args.parts_per_gpu} ({args.parts_per_gpu} per GPU)"
                                       if world > 1 else
                                       f"1 GPU, {parts} concurrent in-GPU partitions (paper's scheme)" if parts > 1
                                       else "1 GPU, sequential RGF"),
                       "l2": "inputs 32 GiB >> 126 MB L2 (no flush needed)" if args.workload == "cfg4" else "inputs > L2"},
            # executed = the flops this implementation performs (re-associated
            # products); the reference's own op inventory for the
            # same solve is flops_reference_inventory.
            "fp64_tflops_step": achieved_step,
            "pct_fp64_peak_step": 100.0 * achieved_step / (peak * world),  # of the N-GPU aggregate peak
            "flops_per_step": executed,
            "flops_reference_inventory": F,
            "effective_tflops_reference_inventory": F / (ms * 1e-3) / 1e12,
            "roofline": {"bound": "tensor", "kernel": "zgemm3m_kernel (3M complex GEMM, DMMA + TMA)",
                         "achieved": gemm_tflops,
                         "peak": peak, "unit": "TFLOP/s", "frac": (gemm_tflops / peak) if gemm_tflops else None,
                         "achieved_basis": "EXECUTED tensor-pipe flops (3M: 6MNK per complex product; exact "
                                           "real-embedding kernel for small products: 8MNK) of all its launches in "
                                           "one instrumented step / union of their CUDA-event spans (busy time)",
                         "frac_executed": (gemm_tflops / peak) if gemm_tflops else None,
                         # the same rate per phase (rank 0's profiled step): in the backward the GEMM
                         # is the bottleneck; the forward is bound by the Schur chains (block inverses)
                         "by_phase": by_phase,
                         "frac_executed_backward": (by_phase["backward"]["gemm_executed_tflops"] / peak
                                                    if by_phase and by_phase["backward"]["gemm_executed_tflops"]
                                                    else None),
                         "achieved_algorithmic": gemm_tflops_alg,
                         "achieved_algorithmic_basis": "8MNK per complex product (the reference's counting) over "
                                                       "the same busy time; exceeds the DMMA peak by up to 4/3 "
                                                       "because the 3M form executes 3/4 of it",
                         "frac_reference_inventory": F / (ms * 1e-3) / 1e12 / (peak * world),
                         "frac_reference_inventory_basis": "reference op inventory (SURVEY 8(d), 8MNK, sequential) "
                                                           "/ step time / (peak x GPUs); > 1 because this "
                                                           "implementation executes far fewer flops",
                         "executed_over_inventory": executed / F,
                         "algorithmic_over_inventory": algorithmic / F,
                         # DRAM bytes per launch of this kernel from one ncu --set full capture of its
                         # launches in the two-lane cfg4-shaped step (profiles/ncu_gemm3m_step_r02.json)
                         "traffic": ncu["mean"]["dram_bytes"] if ncu else None,
                         "traffic_source": ("ncu --set full, " + ncu["target"]) if ncu else None,
                         # every operand read once + outputs written once, live over this step's launches
                         "compulsory_bytes_per_launch": (prof.gemm_bytes / prof.gemm_launches
                                                         if prof.gemm_launches else None),
                         "traffic_over_compulsory": (ncu["mean"]["dram_bytes"] / (prof.gemm_bytes / prof.gemm_launches)
                                                     if ncu and prof.gemm_launches else None),
                         "ncu_dmma_pct_of_peak_active": ncu["mean"]["dmma_inst_pct_of_peak_active"] if ncu else None,
                         "peak_source": peak_src,
                         # busy share of the instrumented step (rank 0)
                         "share_of_step": prof.gemm_busy_ms / prof_ms if prof_ms else None,
                         "inverse_busy_ms_per_step": prof.inverse_busy_ms,
                         "gemm_launches_per_step": prof.gemm_launches},
            "phases_ms": phases,
            "rank_phases_ms": rank_phases,
            "step_ms": step_ms,
            "partition_sizes": ([hi - lo for lo, hi in solver.plan.ranges] if world > 1 else None),
            "partition_plan": (("B200-measured per-block costs (end, middle) = " + str(plan_costs)) if world > 1
                               and plan_costs else ("reference plan_partitions" if world > 1 else None)),
            "value_sequential_rgf_ms": seq_ms,
            "value_general_b_ms": other_b.get("general"),
            "value_antihermitian_b_ms": other_b.get("antihermitian"),
            "flops_per_step_algorithmic": algorithmic,
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "input_generation_s": t_gen,
            "config5": cfg5,
        }
        emit(line)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
