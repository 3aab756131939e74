#!/usr/bin/env python
"""The CPU reference baseline, full protocol:
the UNMODIFIED reference btasel (baseline/_ref, tools/stage_reference.sh)
solve_selected on the bench-protocol inputs of config 4's block shapes
(b=512, a=256) at n in {32, 64, 128}, with BLAS threads = all host cores and
= 1, a least-squares line t = t0 + s*n per thread count, extrapolated to
n=1024 (linearity is reference acceptance criterion 7); the faster thread
count is the baseline.  Runs on the GPU box's host (config 4 needs ~104 GiB,
so the full size is not run).  Prints one JSON object (commit under
profiles/cpu_protocol_r02.json).

    python tools/cpu_protocol.py [--ns 32,64,128] [--threads all,1]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (host_info, reference_impl, set_host_blas_threads)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="32,64,128")
    ap.add_argument("--threads", default="all,1")
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--b", type=int, default=512)
    ap.add_argument("--a", type=int, default=256)
    args = ap.parse_args()
    ref, kind = bench.reference_impl()
    ns = [int(x) for x in args.ns.split(",")]
    out = {"kind": kind, "workload": f"config 4 block shapes b={args.b}, a={args.a}; extrapolated to n={args.n}",
           "host": bench.host_info(), "runs": {}, "fit": {}}
    for th in args.threads.split(","):
        t = bench.host_cores() if th == "all" else int(th)
        pts = []
        for n in ns:
            A = ref.generate_dd_bta(n, args.b, args.a, seed=0)
            B = ref.hermitianize(ref.generate_dd_bta(n, args.b, args.a, seed=1))
            bench.set_host_blas_threads(t)
            t0 = time.perf_counter()
            ref.solve_selected(A, B, "siq")
            pts.append((n, time.perf_counter() - t0))
            del A, B
            print(f"threads={t} n={n}: {pts[-1][1]:.1f} s", file=sys.stderr, flush=True)
        k = len(pts)
        mx = sum(p[0] for p in pts) / k
        my = sum(p[1] for p in pts) / k
        slope = sum((p[0] - mx) * (p[1] - my) for p in pts) / sum((p[0] - mx) ** 2 for p in pts)
        t0 = my - slope * mx
        out["runs"][str(t)] = [{"n": n, "s": round(s, 3)} for n, s in pts]
        out["fit"][str(t)] = {"t0_s": t0, "s_per_block": slope, "extrapolated_ms": (t0 + slope * args.n) * 1e3}
    best = min(out["fit"], key=lambda k: out["fit"][k]["extrapolated_ms"])
    out["value_ms"] = out["fit"][best]["extrapolated_ms"]
    out["value_threads"] = int(best)
    bench.emit(out)  # bench.py routes fd 1 to stderr; emit() writes to the real stdout


if __name__ == "__main__":
    main()
