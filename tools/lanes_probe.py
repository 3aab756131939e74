"""Time cfg4 solve: sequential vs the 2-partition scheme run concurrently on one GPU."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2601_04904_b200 as bs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
A = bs.generate_dd_bta_device(n, 512, 256, seed=0)
B = bs.hermitianize_device(bs.generate_dd_bta_device(n, 512, 256, seed=1))
for parts in (1, 2, 1, 2):
    t = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = bs.dist_solve(A, B, num_parts=parts, mode="siq", timings=t)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(parts, f"{dt*1e3:.1f} ms", {k: round(v * 1e3, 1) for k, v in t.items()}, flush=True)
    del sol
ref = bs.dist_solve(A, B, num_parts=1, mode="siq")
got = bs.dist_solve(A, B, num_parts=2, mode="siq")
err = max((torch.linalg.norm(g - r) / torch.linalg.norm(r)).item() for X, Y in ((got.x_a, ref.x_a), (got.x_b, ref.x_b))
          for g, r in zip(X.diag[::97], Y.diag[::97]))
print("max diag block rel err (P=2 vs P=1):", err)
