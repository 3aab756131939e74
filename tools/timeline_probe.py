"""Per-launch timeline of one cfg4 solve (BSEL_PROFILE_DUMP): per stream busy
time, inverse durations, gaps on the chain stream.  argv: parts [n]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200 import _native  # noqa: E402

parts = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
mode = sys.argv[3] if len(sys.argv) > 3 else "siq"
path = os.environ.setdefault("BSEL_PROFILE_DUMP", "/tmp/timeline.csv")
if os.environ.get("PROBE_AVOID_SMS"):  # one lane: aux levels leave SMs to the chain (DistSolver default)
    _native.Context.get(torch.cuda.current_device()).set_aux_avoid_sms(int(os.environ["PROBE_AVOID_SMS"]))
A = bs.generate_dd_bta_device(n, 512, 256, seed=0)
B = bs.hermitianize_device(bs.generate_dd_bta_device(n, 512, 256, seed=1))
Bm = B if mode == "siq" else None
for _ in range(2):
    bs.solve_selected(A, Bm, mode, partitions=parts)
torch.cuda.synchronize()
lib = _native.load_library()
prof = _native.Profile()
t = {}
lib.bsel_profile_begin()
bs.solve_selected(A, Bm, mode, partitions=parts, timings=t)
lib.bsel_profile_end(prof)
print("phases ms", {k: round(v * 1e3, 1) for k, v in t.items()})
rows = [line.strip().split(",") for line in open(path)]
rows = [(int(r[0]), r[1], float(r[2]), float(r[3]), float(r[4])) for r in rows]
streams = {}
for k, s, a, b, f in rows:
    streams.setdefault(s, []).append((a, b, k, f))
t0 = min(r[2] for r in rows)
t1 = max(r[3] for r in rows)
print(f"span {t1 - t0:.1f} ms, launches {len(rows)}")
for s, v in streams.items():
    v.sort()
    busy = sum(b - a for a, b, _, _ in v)
    inv = [b - a for a, b, k, _ in v if k == 1]
    gem = [(b - a, f) for a, b, k, f in v if k == 0]
    gaps = [v[i + 1][0] - v[i][1] for i in range(len(v) - 1)]
    gaps = [g for g in gaps if g > 0]
    line = f"stream {s}: launches {len(v)} busy {busy:.1f} ms, gaps total {sum(gaps):.1f} ms"
    if inv:
        inv.sort()
        line += (f"; inverses {len(inv)} total {sum(inv):.1f} ms, median {inv[len(inv)//2]*1e3:.0f} us, "
                 f"p10 {inv[len(inv)//10]*1e3:.0f} us p90 {inv[9*len(inv)//10]*1e3:.0f} us")
    if gem:
        fl = sum(f for _, f in gem)
        line += f"; gemm {len(gem)} launches {sum(d for d, _ in gem):.1f} ms, {fl/1e12:.2f} TFLOP"
    print(line)
