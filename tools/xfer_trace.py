"""One streamed solve with BSEL_XFER_TRACE=1 (chunk arrival vs chain)."""
import os
import sys

os.environ["BSEL_XFER_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2601_04904_b200 as bs  # noqa: E402

n, b, a = 1024, 512, 256
A = bs.generate_dd_bta_device(n, b, a, seed=0)
B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1))
hA = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
hB = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
A.copy_to_host(hA)
B.copy_to_host(hB)
del A, B
torch.cuda.empty_cache()
hX = (bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False), bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False))
for _ in range(2):
    bs.solve_selected(hA, hB, "siq", out=hX)
