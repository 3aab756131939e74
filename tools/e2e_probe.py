"""Where does the end-to-end time go?  Phase times of a streamed host-I/O
solve vs a device-resident solve, plus raw pinned H2D/D2H bandwidth."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200 import rgf  # noqa: E402

n, b, a = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 512, 256)))
dev = torch.device("cuda:0")
A = bs.generate_dd_bta_device(n, b, a, seed=0)
B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1))
hA = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
hB = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
A.copy_to_host(hA)
B.copy_to_host(hB)
torch.cuda.synchronize()


def ev_time(fn, reps=2):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


h2d = ev_time(lambda: A.copy_from_host(hA, non_blocking=True))
d2h = ev_time(lambda: A.copy_to_host(hA, non_blocking=True))
gb = hA.nbytes / 1e9
print(f"pinned H2D {gb:.1f} GB: {h2d:.1f} ms = {gb / h2d * 1e3:.1f} GB/s; D2H {d2h:.1f} ms = {gb / d2h * 1e3:.1f} GB/s")

XA, XB = bs.DeviceBta.empty(n, b, a, dev), bs.DeviceBta.empty(n, b, a, dev)
t = {}
dms = ev_time(lambda: bs.solve_selected(A, B, "siq", out=(XA, XB), timings=t))
print(f"device-resident: {dms:.1f} ms; phases {({k: round(v * 1e3, 1) for k, v in t.items()})}")
runner = next(iter(rgf._PARTITIONED.values()))
print("  device phases", {k: round(v * 1e3, 1) for k, v in runner.phase_seconds().items()})
del XA, XB, A, B
torch.cuda.empty_cache()
hXA = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
hXB = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
for chunk in (8, 4, 16, 32):
    os.environ["BSEL_STREAM_CHUNK"] = str(chunk)
    t0 = time.perf_counter()
    ms = ev_time(lambda: bs.solve_selected(hA, hB, "siq", out=(hXA, hXB)))
    runner = [r for k, r in rgf._PARTITIONED.items()][0]
    print(f"streamed chunk={chunk}: {ms:.1f} ms; phases",
          {k: round(v * 1e3, 1) for k, v in runner.phase_seconds().items()},
          f"wall {(time.perf_counter() - t0) / 3 * 1e3:.0f} ms/call")
