#!/bin/bash
# ncu --set full of the dataflow block inverse alone (tools/inv_probe.py, n=512, 64 CTAs),
# after the same command exited 0 without ncu; summary -> gpurun_out/ncu_inverse_df.json
set -e
timeout 300 python tools/inv_probe.py 512
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dataflow_gj -s 2 -c 2 \
  -o gpurun_out/ncu_df -f python tools/inv_probe.py 512 > gpurun_out/ncu_df.log 2>&1
ncu -i gpurun_out/ncu_df.ncu-rep --page raw --csv > gpurun_out/ncu_df_raw.csv
python tools/ncu_inverse_summary.py gpurun_out/ncu_df_raw.csv gpurun_out/ncu_inverse_df.json \
  "tools/inv_probe.py 512 (512x512 DD block, alone): dataflow_gj_kernel launches 3-4, ncu --set full, serialized"
ncu -i gpurun_out/ncu_df.ncu-rep --page source --csv > gpurun_out/ncu_df_source.csv 2>/dev/null || true
rm -f gpurun_out/ncu_df.ncu-rep
