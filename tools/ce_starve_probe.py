"""Probe: does a 4-byte D2H on one stream wait behind a 16 GiB D2H queued on
another stream (one call, or 32 MiB pieces)?  Host wall time of the small
read (copy + stream sync)."""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200.energy import HostEnergySweep  # noqa: E402

n, b, a = 1024, 512, 256
dev = torch.device("cuda", 0)
D = bs.DeviceBta.empty(n, b, a, dev, zero=False)
H = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
hflag = torch.zeros(1, dtype=torch.int32).pin_memory()
big, small = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
mapped = torch.zeros(1, dtype=torch.int32).pin_memory()  # kernel writes it through a device view? (UVA)
v = (flag + 1).sum()  # warm the kernels
torch.cuda.synchronize()
ev = torch.cuda.Event()
for mode in ("whole", "chunked", "kernel-read", "kernel-event", "whole"):
    torch.cuda.synchronize()
    with torch.cuda.stream(big):
        if mode == "chunked":
            HostEnergySweep._chunked(H, D, True)
        else:
            D.copy_to_host(H, non_blocking=True)
    time.sleep(0.02)
    t0 = time.perf_counter()
    with torch.cuda.stream(small):
        if mode == "kernel-event":
            v = (flag + 1).sum()
            ev.record(small)
            ev.synchronize()
        elif mode == "kernel-read":
            v = (flag + 1).sum()  # kernel only, no copy: baseline for a launch + sync
            small.synchronize()
        else:
            hflag.copy_(flag, non_blocking=True)
            small.synchronize()
    t1 = time.perf_counter()
    big.synchronize()
    t2 = time.perf_counter()
    print(f"{mode}: small read waited {1e3 * (t1 - t0):.1f} ms; big copy done after {1e3 * (t2 - t0):.1f} ms",
          flush=True)
