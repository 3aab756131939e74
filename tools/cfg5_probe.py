"""Config 5 (n=256, b=1024, a=256) energy sweep on cuda:0: ms per energy
(1 warm-up energy, argv[1] timed energies, device-timed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_04904_b200 as bs  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sweep = bs.EnergySweep(256, 1024, 256, "siq", device=torch.device("cuda:0"))
sweep.run([0])
torch.cuda.synchronize()
out = []
for rep in range(3):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    sweep.run(list(range(1 + rep * k, 1 + (rep + 1) * k)))
    e.record()
    torch.cuda.synchronize()
    out.append(round(s.elapsed_time(e) / k, 1))
print(f"cfg5 ms/energy {out} (overlap {sweep.overlap}, dataflow {os.environ.get('BSEL_INV_DATAFLOW', '1')})")
