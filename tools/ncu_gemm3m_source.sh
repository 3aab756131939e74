#!/bin/bash
# ncu --set full with source (SASS) of one 3M GEMM launch on the backward level
# bwd_L1_12p (tools/gemm3m_micro profiling mode, cfg 14 = 64x32 / BK 32);
# exports raw + source CSVs to gpurun_out/.
set -e
./tools/gemm3m_micro 0 14 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zgemm3m -s 2 -c 1 \
  -o gpurun_out/ncu_g3m -f ./tools/gemm3m_micro 0 14 3 > gpurun_out/ncu_g3m.log 2>&1
ncu -i gpurun_out/ncu_g3m.ncu-rep --page raw --csv > gpurun_out/ncu_g3m_raw.csv
ncu -i gpurun_out/ncu_g3m.ncu-rep --page source --csv > gpurun_out/ncu_g3m_source.csv
ncu -i gpurun_out/ncu_g3m.ncu-rep --page details --csv > gpurun_out/ncu_g3m_details.csv
rm -f gpurun_out/ncu_g3m.ncu-rep
