#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -o gpurun_out/r2_dec1 \
  python tools/op_profile.py --op decode --batch 1 > gpurun_out/r2_dec1.log 2>&1
python tools/ncu_summary.py gpurun_out/r2_dec1.ncu-rep > gpurun_out/r2_dec1_summary.txt 2>&1
ncu -i gpurun_out/r2_dec1.ncu-rep --page source --csv --kernel-name regex:topk_select > gpurun_out/r2_dec1_select_source.csv 2>&1
ncu -i gpurun_out/r2_dec1.ncu-rep --page source --csv --kernel-name regex:topk_hist > gpurun_out/r2_dec1_hist_source.csv 2>&1
rm -f gpurun_out/r2_dec1.ncu-rep
