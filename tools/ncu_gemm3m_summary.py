#!/usr/bin/env python
"""Summarise an ncu --set full capture of zgemm3m_kernel launches (one JSON):
per launch duration, DRAM bytes, DMMA (tensor FP64) pipe activity, shared
bank conflicts, and the mean over the captured launches.
    python tools/ncu_gemm3m_summary.py gpurun_out/prof_step64.ncu-rep "target description"
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
target = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
idx = {k: i for i, k in enumerate(h)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6, "nsecond": 1e-9, "ns": 1e-9, "msecond": 1e-3, "ms": 1e-3}


def val(r, k):
    x = float(r[idx[k]].replace(",", ""))
    return x * scale.get(units[idx[k]], 1.0)


launches = []
for r in rows[2:]:
    if "zgemm3m" not in r[idx["Kernel Name"]]:
        continue
    d = {
        "time_s": val(r, "gpu__time_duration.sum"),
        "dram_read_bytes": val(r, "dram__bytes_read.sum"),
        "dram_write_bytes": val(r, "dram__bytes_write.sum"),
        "dmma_inst_pct_of_peak_active": val(r, "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
        "fp64_tensor_ops_pct_of_peak_elapsed": val(r, "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed"),
        "fp64_tensor_ops": val(r, "sm__ops_path_tensor_src_fp64.sum"),
        "grid": int(val(r, "launch__grid_size")),
        "registers": int(val(r, "launch__registers_per_thread")),
        "smem_ld_bank_conflicts": val(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
    }
    d["dram_bytes"] = d["dram_read_bytes"] + d["dram_write_bytes"]
    d["executed_tflops"] = d["fp64_tensor_ops"] / d["time_s"] / 1e12 if d["time_s"] else None  # ops = flops (peak 128/clk/SM)
    launches.append(d)
n = len(launches)
mean = {k: sum(l[k] for l in launches) / n for k in launches[0] if isinstance(launches[0][k], (int, float))}
print(json.dumps({"target": target, "launches": n, "mean": mean, "per_launch": launches}, indent=1))
