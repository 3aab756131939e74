"""Target for the launch-list capture (ncu --metrics gpu__time_duration.sum):
one cfg4-shaped SI+SQ solve (b=512, a=256) with n=32 blocks through the
bench path (2 in-GPU partitions), after 2 warm-up solves."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_04904_b200 as bs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
A = bs.generate_dd_bta_device(n, 512, 256, seed=0)
B = bs.hermitianize_device(bs.generate_dd_bta_device(n, 512, 256, seed=1))
XA, XB = bs.DeviceBta.empty(n, 512, 256, A.device), bs.DeviceBta.empty(n, 512, 256, A.device)
for _ in range(3):
    bs.solve_selected(A, B, "siq", out=(XA, XB), partitions=2)
torch.cuda.synchronize()
print("ok")
