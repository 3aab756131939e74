"""Summarize `ncu -i rep --page raw --csv` of block-inverse launches (one row
per launch): duration, grid, registers, DMMA pipe activity, FP64 tensor
share of peak, DRAM bytes, warps active, top stall reasons (per issue).
usage: ncu_inverse_summary.py raw.csv out.json target-description"""
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__registers_per_thread",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]
pre = "smsp__average_warps_issue_stalled_"
out = []
for r in data:
    d = {}
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            d[w] = f"{r[i]} {units[i]}".strip()
    st = []
    for i, h in enumerate(hdr):
        if h.startswith(pre) and h.endswith("_per_issue_active.ratio"):
            try:
                st.append((h[len(pre):-len("_per_issue_active.ratio")], float(r[i].replace(",", ""))))
            except ValueError:
                pass
    d["top_stalls"] = sorted(st, key=lambda x: -x[1])[:6]
    out.append(d)
json.dump({"target": sys.argv[3], "launches": out}, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1)[:3000])
