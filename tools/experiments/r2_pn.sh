#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/r2_pfn_b1 python tools/op_profile.py --op pfn --batch 1 > gpurun_out/r2_pfn_b1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/r2_pfn_b32 python tools/op_profile.py --op pfn --batch 32 > gpurun_out/r2_pfn_b32.log 2>&1
