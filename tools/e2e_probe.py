"""Probe: HostEnergySweep at config 4 shapes, out_slots 1 vs 2 (pipelined
end-to-end ms per energy point, allocator retries, free device memory)."""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_04904_b200 as bs  # noqa: E402

n, b, a = 1024, 512, 256
slots = int(sys.argv[1]) if len(sys.argv) > 1 else 2
k = int(sys.argv[2]) if len(sys.argv) > 2 else 6
dev = torch.device("cuda", 0)
A = bs.generate_dd_bta_device(n, b, a, seed=0, device=dev)
B = bs.hermitianize_device(bs.generate_dd_bta_device(n, b, a, seed=1, device=dev))
hA = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
hB = bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False)
A.copy_to_host(hA)
B.copy_to_host(hB)
del A, B
torch.cuda.empty_cache()
hX = (bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False), bs.BtaMatrix.zeros(n, b, a, pinned=True, zero=False))
sweep = bs.HostEnergySweep(n, b, a, "siq", out_slots=slots)
print("free GiB after sweep buffers", torch.cuda.mem_get_info()[0] / 2**30, flush=True)
sweep.run([(hA, hB)] * 2, [hX] * 2)
torch.cuda.synchronize()
r0 = torch.cuda.memory_stats().get("num_alloc_retries", 0)
for kk in (1, k):
    t0 = time.perf_counter()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    sweep.run([(hA, hB)] * kk, [hX] * kk)
    e.record()
    torch.cuda.synchronize()
    torch.cuda.synchronize()
    print("  solve-done times (ms from start):", [round(s.elapsed_time(d), 1) for d in sweep.done_events])
    print(f"out_slots={slots} K={kk}: {s.elapsed_time(e) / kk:.1f} ms/energy (wall {1e3 * (time.perf_counter() - t0) / kk:.1f})",
          flush=True)
print("alloc retries during timed runs", torch.cuda.memory_stats().get("num_alloc_retries", 0) - r0)
print("free GiB", torch.cuda.mem_get_info()[0] / 2**30)
