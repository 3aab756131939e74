"""Per-stream statistics of a BSEL_PROFILE_DUMP timeline (kind, stream, start,
end, flops, exec_flops), split at the last block inverse (forward / backward).
argv: dump files.  The chain stream is the one that launches the inverses."""
import sys


def stats(path):
    rows = []
    for line in open(path):
        p = line.strip().split(",")
        if len(p) >= 6:
            rows.append((int(p[0]), p[1], float(p[2]), float(p[3]), float(p[4]), float(p[5])))
    inv_end = max(r[3] for r in rows if r[0] == 1)
    t0 = min(r[2] for r in rows)
    chains = {r[1] for r in rows if r[0] == 1}
    print(f"{path}: {len(rows)} launches, forward span {inv_end - t0:.1f} ms, step span "
          f"{max(r[3] for r in rows) - t0:.1f} ms")
    for s in sorted({r[1] for r in rows}):
        v = sorted((r for r in rows if r[1] == s and r[3] <= inv_end), key=lambda r: r[2])
        if not v:
            continue
        busy = sum(r[3] - r[2] for r in v)
        gaps = [v[i + 1][2] - v[i][3] for i in range(len(v) - 1)]
        big = sorted(g for g in gaps if g > 0.02)
        inv = sorted(r[3] - r[2] for r in v if r[0] == 1)
        gem = [r for r in v if r[0] == 0]
        line = (f"  fwd stream {s}{' (chain)' if s in chains else ''}: {len(v)} launches, busy {busy:.1f} ms "
                f"({busy / (inv_end - t0):.0%}), gaps>20us {len(big)} total {sum(big):.1f} ms")
        if inv:
            line += (f"; inverses {len(inv)} {sum(inv):.1f} ms median {inv[len(inv) // 2] * 1e3:.0f} us")
        if gem:
            gt = sorted(r[3] - r[2] for r in gem)
            line += (f"; gemm {len(gem)} {sum(gt):.1f} ms median {gt[len(gt) // 2] * 1e3:.0f} us, "
                     f"{sum(r[5] for r in gem) / 1e12:.2f} TFLOP exec")
        print(line)


for f in sys.argv[1:]:
    stats(f)
