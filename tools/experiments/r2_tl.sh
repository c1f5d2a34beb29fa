#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
PMX_LIB=paper_2601_12638_b200/libpmx_trace.so timeout 300 python tools/b1_timeline.py > gpurun_out/r2_tl_mixed.log 2>&1
PMX_LIB=paper_2601_12638_b200/libpmx_trace.so PMX_NECK_STREAM=0 timeout 300 python tools/b1_timeline.py > gpurun_out/r2_tl_mixed_noneck.log 2>&1
