"""Forward/backward phase times of cfg4 in si and siq modes, 1 and 2 lanes
(is the forward chain-bound?)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2601_04904_b200 as bs  # noqa: E402

n, b, a = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1024, 512, 256)))
A = bs.generate_dd_bta_device(n, b, a, seed=0)
B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1))
for mode in ("si", "siq"):
    for parts in (1, 2):
        t = {}
        for _ in range(2):
            bs.solve_selected(A, B if mode == "siq" else None, mode, partitions=parts, timings=t)
        torch.cuda.synchronize()
        print(mode, "parts", parts, {k: round(v * 1e3, 1) for k, v in t.items()}, flush=True)
