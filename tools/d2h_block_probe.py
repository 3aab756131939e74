"""Probe: does DeviceBta.copy_to_host(non_blocking=True) block the host
thread?  Host-side call duration vs cudaMemcpyAsync (cuda-python) for one
config-4 BtaMatrix (16 GiB) on a side stream."""

import os
import sys
import time

import torch
from cuda.bindings import runtime as rt

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04904_b200 as bs  # noqa: E402

n, b, a = 1024, 512, 256
dev = torch.device("cuda", 0)
D = bs.DeviceBta.empty(n, b, a, dev, zero=False)
H = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
s = torch.cuda.Stream(dev)
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        D.copy_to_host(H, non_blocking=True)
    t1 = time.perf_counter()
    s.synchronize()
    t2 = time.perf_counter()
    print(f"torch copy_ D2H: call {1e3 * (t1 - t0):.1f} ms, done {1e3 * (t2 - t0):.1f} ms", flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        D.copy_from_host(H, non_blocking=True)
    t1 = time.perf_counter()
    s.synchronize()
    t2 = time.perf_counter()
    print(f"torch copy_ H2D: call {1e3 * (t1 - t0):.1f} ms, done {1e3 * (t2 - t0):.1f} ms", flush=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k, arr in H.stacked().items():
        if arr.size:
            t = getattr(D, k)
            err, = rt.cudaMemcpyAsync(arr.ctypes.data, t.data_ptr(), arr.nbytes,
                                      rt.cudaMemcpyKind.cudaMemcpyDeviceToHost, s.cuda_stream)
            assert err == rt.cudaError_t.cudaSuccess, err
    t1 = time.perf_counter()
    s.synchronize()
    t2 = time.perf_counter()
    print(f"cudaMemcpyAsync D2H: call {1e3 * (t1 - t0):.1f} ms, done {1e3 * (t2 - t0):.1f} ms", flush=True)
