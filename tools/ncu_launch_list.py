#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel
(launches, total, share, average) as a markdown table.
    python tools/ncu_launch_list.py gpurun_out/launches.csv "title" > profiles/ncu_launches_rNN.md
"""
import collections
import csv
import sys

path, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = []
with open(path) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1e3 if unit in ("nsecond", "ns") else v if unit in ("usecond", "us") else v * 1e3
    name = r["Kernel Name"]
    name = name.split("(")[0] if "<" not in name else name[: name.find(">(") + 1]
    rows.append((name, us))
tot = sum(u for _, u in rows)
agg = collections.defaultdict(lambda: [0, 0.0])
for n, u in rows:
    agg[n][0] += 1
    agg[n][1] += u
print(f"# ncu launch list — {title}\n")
print("Per-launch times are cold-cache and serialised (no stream overlap): compare SHARES, not absolutes.\n")
print("| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
for n, (c, u) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"| `{n[-90:]}` | {c} | {u:.1f} | {100 * u / tot:.1f}% | {u / c:.1f} |")
print(f"\nTotal: {len(rows)} launches, {tot:.1f} us.")
