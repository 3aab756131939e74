#!/usr/bin/env python
"""Kernel microbenchmarks (B200): grouped DMMA ZGEMM throughput, block-inverse
latency, sweep phase split.  Prints one JSON object.  Timings: CUDA events on
the launching stream after warm-up."""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200 import _native  # noqa: E402


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    out = {}
    dev = torch.device("cuda", 0)
    c = lambda *s: torch.randn(*s, dtype=torch.complex128, device=dev)  # noqa: E731
    for m, k, n, ta, tb in ((512, 512, 512, 0, 0), (512, 512, 512, 1, 0), (512, 512, 512, 0, 1),
                            (1024, 1024, 1024, 0, 0), (2048, 2048, 2048, 0, 0), (256, 512, 512, 0, 0)):
        a = c(k, m) if ta else c(m, k)
        b = c(n, k) if tb else c(k, n)
        ms = ev_time(lambda: bs.block_multiply_acc(None, a, b, trans_a=bool(ta), trans_b=bool(tb)), 10)
        out[f"zgemm_{m}x{k}x{n}_{'HN'[not ta]}{'HN'[not tb]}_tflops"] = 8.0 * m * k * n / ms / 1e9
    for n in (64, 128, 256, 512, 1024):
        x = c(n, n) + 3 * n * torch.eye(n, dtype=torch.complex128, device=dev)
        bs.block_inverse(x)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 20
        for _ in range(reps):
            bs.block_inverse(x)
        torch.cuda.synchronize()
        out[f"inverse_{n}_us_wall"] = (time.perf_counter() - t0) / reps * 1e6
    # profile of one cfg4-shaped solve (n=64): per-kernel totals and phases
    A = bs.generate_dd_bta_device(64, 512, 256, seed=0)
    B = bs.hermitianize_device(bs.generate_dd_bta_device(64, 512, 256, seed=1))
    t = {}
    bs.solve_selected(A, B, timings=t)
    bs.solve_selected(A, B, timings=t)
    out["cfg4_n64_forward_ms"] = t["forward"] * 1e3
    out["cfg4_n64_backward_ms"] = t["backward"] * 1e3
    lib = _native.load_library()
    prof = _native.Profile()
    lib.bsel_profile_begin()
    bs.solve_selected(A, B)
    lib.bsel_profile_end(prof)
    out["cfg4_n64_gemm_tflops"] = prof.gemm_flops / prof.gemm_ms / 1e9
    out["cfg4_n64_inverse_ms_each"] = prof.inverse_ms / max(prof.inverse_calls, 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
