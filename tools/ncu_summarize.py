"""Summarize an `ncu -i rep --page raw --csv` export (one row per launch):
per-launch DRAM bytes, durations, tensor/DMMA pipe activity.  Run on the GPU
box next to the capture (the .ncu-rep itself is too large to bring back).
usage: ncu_summarize.py raw.csv out.json [algorithmic_flops_total compulsory_bytes_total]"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def num(r, name):
    try:
        return float(r[col[name]].replace(",", ""))
    except (KeyError, ValueError):
        return None


def scale(name):
    u = units[col[name]] if name in col else ""
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
            "msecond": 1e-3, "second": 1.0, "us": 1e-6, "ns": 1e-9, "ms": 1e-3, "s": 1.0}.get(u, 1.0)


keys = [h for h in hdr if any(s in h for s in ("tensor", "dmma", "fp64", "dram__bytes", "gpu__time_duration",
                                               "launch__grid_size", "sm__throughput", "registers"))]
out = {"launches": len(data), "metrics_seen": keys}
tot = {}
for name in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
    if name in col:
        tot[name] = sum((num(r, name) or 0.0) for r in data) * scale(name)
out["time_s_sum"] = tot.get("gpu__time_duration.sum")
if "dram__bytes_read.sum" in tot:
    out["dram_read_bytes_per_launch"] = tot["dram__bytes_read.sum"] / len(data)
    out["dram_write_bytes_per_launch"] = tot["dram__bytes_write.sum"] / len(data)
    out["dram_bytes_per_launch"] = out["dram_read_bytes_per_launch"] + out["dram_write_bytes_per_launch"]
# time-weighted pipe activity for every pct metric of the tensor / fp64 pipes
tcol = "gpu__time_duration.sum"
if tcol in col:
    w = [num(r, tcol) or 0.0 for r in data]
    W = sum(w) or 1.0
    for k in keys:
        if "pct" in k:
            vals = [num(r, k) for r in data]
            if all(v is not None for v in vals):
                out["tw_" + k] = sum(v * x for v, x in zip(vals, w)) / W
if len(sys.argv) > 4:
    flops, comp = float(sys.argv[3]), float(sys.argv[4])
    out["algorithmic_flops_per_launch"] = flops / len(data)
    out["compulsory_bytes_per_launch"] = comp / len(data)
    if "dram_bytes_per_launch" in out:
        out["traffic_over_compulsory"] = out["dram_bytes_per_launch"] / out["compulsory_bytes_per_launch"]
        out["flop_per_dram_byte"] = out["algorithmic_flops_per_launch"] / out["dram_bytes_per_launch"]
    if out.get("time_s_sum"):
        out["achieved_tflops_ncu_time"] = flops / out["time_s_sum"] / 1e12
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "metrics_seen"}, indent=1))
