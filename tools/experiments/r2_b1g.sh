#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_b1g.log
: > $O
for v in 1 0; do
  PMX_GATHER=$v PMX_LIB=paper_2601_12638_b200/libpmx_trace.so timeout 300 python tools/b1_timeline.py > gpurun_out/r2_tl_g$v.log 2>&1
  head -6 gpurun_out/r2_tl_g$v.log >> $O
done
for op in pillarize pfn decode records; do
  for b in 1; do
    timeout 300 python tools/op_profile.py --op $op --batch $b --time 2>&1 | tail -1 >> $O
  done
done
