#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  python tools/op_profile.py --op decode --batch 1 > gpurun_out/r2_dec_ncu.csv 2>gpurun_out/r2_dec_ncu.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  python tools/op_profile.py --op pillarize --batch 1 > gpurun_out/r2_pz_ncu.csv 2>gpurun_out/r2_pz_ncu.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  python tools/op_profile.py --op pfn --batch 1 > gpurun_out/r2_pfn_ncu.csv 2>gpurun_out/r2_pfn_ncu.err
