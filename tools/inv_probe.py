"""Run the block inverse on a 512 (or argv[1]) DD matrix a few times (ncu target)."""
import sys
import torch
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2601_04904_b200 as bs  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
x = torch.randn(n, n, dtype=torch.complex128, device="cuda") + 3 * n * torch.eye(n, dtype=torch.complex128, device="cuda")
for _ in range(5):
    bs.block_inverse(x)
torch.cuda.synchronize()
print("ok", n)
