"""Pinned H2D throughput: one big copy vs 32 MiB chunks on one / two streams,
alone and next to a DMMA-heavy kernel load (what the streamed forward sees)."""
import torch

GB = 1 << 30
total = 16 * GB
piece = 32 << 20
host = torch.empty(total // 16, dtype=torch.complex128, pin_memory=True)
dev = torch.empty_like(host, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run(streams, load=False):
    torch.cuda.synchronize()
    ls = torch.cuda.Stream()
    if load:
        x = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda")
        with torch.cuda.stream(ls):
            for _ in range(40):
                x = x @ x * 1e-3
    s, e = ev(), ev()
    s.record()
    ss = [torch.cuda.Stream() for _ in range(streams)]
    for st in ss:
        st.wait_stream(torch.cuda.current_stream())
    n = total // piece
    per = piece // 16
    for i in range(n):
        st = ss[i % streams]
        with torch.cuda.stream(st):
            dev[i * per:(i + 1) * per].copy_(host[i * per:(i + 1) * per], non_blocking=True)
    for st in ss:
        torch.cuda.current_stream().wait_stream(st)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    return total / 1e9 / (ms / 1e3)


big_s, big_e = ev(), ev()
big_s.record()
dev.copy_(host, non_blocking=True)
big_e.record()
torch.cuda.synchronize()
print(f"one copy: {total / 1e9 / (big_s.elapsed_time(big_e) / 1e3):.1f} GB/s")
for streams in (1, 2, 4):
    print(f"32 MiB chunks, {streams} stream(s): {run(streams):.1f} GB/s; with DMMA load: {run(streams, True):.1f} GB/s")
