"""Probe: H2D / D2H / concurrent bandwidth of one config-4 BtaMatrix
(16 GiB) between pinned host BtaMatrix buffers and a DeviceBta, through the
DeviceBta copy helpers (torch copy_) on side streams."""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04904_b200 as bs  # noqa: E402

n, b, a = 1024, 512, 256
dev = torch.device("cuda", 0)
D1 = bs.DeviceBta.empty(n, b, a, dev, zero=False)
D2 = bs.DeviceBta.empty(n, b, a, dev, zero=False)
H1 = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
H2 = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
print("pinned", all(torch.from_numpy(x).is_pinned() for x in H1.stacked().values()))
gib = H1.nbytes / 2**30
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    s1.synchronize()
    s2.synchronize()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def h2d():
    with torch.cuda.stream(s1):
        D1.copy_from_host(H1, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        D2.copy_to_host(H2, non_blocking=True)


for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", lambda: (h2d(), d2h())), ("h2d", h2d), ("d2h", d2h)):
    ms = timed(fn)
    print(f"{name}: {ms:.1f} ms for {gib:.1f} GiB each -> {gib * 2**30 / ms / 1e6:.1f} GB/s per direction", flush=True)
