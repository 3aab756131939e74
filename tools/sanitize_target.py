"""Small solves through every kernel family (sequential + 2 in-GPU
partitions, Hermitian / general B, fused Schur step, SM-avoiding aux levels)
for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_04904_b200 as bs  # noqa: E402
from paper_2601_04904_b200 import _native  # noqa: E402

n, b, a = 8, 72, 20
A = bs.generate_dd_bta(n, b, a, seed=1)
H = bs.hermitianize(bs.generate_dd_bta(n, b, a, seed=2))
G = bs.generate_dd_bta(n, b, a, seed=3)
for B in (H, G):
    bs.solve_selected(A, B, "siq", partitions=1)
    bs.dist_solve(A, B, num_parts=3, mode="siq")
os.environ["BSEL_SCHUR"] = "1"
bs.solve_selected(A, H, "siq", partitions=1)
os.environ.pop("BSEL_SCHUR")
ctx = _native.Context.get(0)
ctx.set_aux_avoid_sms(100)
bs.solve_selected(A, H, "siq", partitions=1)
ctx.set_aux_avoid_sms(0)
torch.cuda.synchronize()
print("ok")
