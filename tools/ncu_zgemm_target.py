"""Target for the roofline-traffic capture: ONE sequential SI+SQ solve at the
config-4 block shapes (b=512, a=256) with n=8 blocks, so every level kind of
the sweeps appears.  Without ncu it writes the live per-launch totals of the
grouped GEMM (algorithmic flops / compulsory bytes / event time) to
gpurun_out/zgemm_target_totals.json; under ncu (-k regex:zgemm_grouped) the
same launches are captured with DRAM byte counters."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200 import _native  # noqa: E402

n, b, a = 8, 512, 256
A = bs.generate_dd_bta_device(n, b, a, seed=0)
B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1))
torch.cuda.synchronize()
lib = _native.load_library()
lib.bsel_profile_begin()
bs.solve_selected(A, B, "siq", partitions=1)
prof = _native.Profile()
lib.bsel_profile_end(ctypes_ref := __import__("ctypes").byref(prof))
tot = {k: getattr(prof, k) for k, _ in _native.Profile._fields_}
if not os.environ.get("NV_COMPUTE_PROFILER_PERFWORKS_DIR") and "ncu" not in os.environ.get("_", ""):
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/zgemm_target_totals.json", "w") as f:
        json.dump({"n": n, "b": b, "a": a, **tot}, f, indent=1)
print(json.dumps(tot))
