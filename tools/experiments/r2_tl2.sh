#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_b1trace.log
: > $O
for op in "conv backbone.blocks.2.3" "conv backbone.blocks.1.3" "conv backbone.blocks.0.3" "conv backbone.blocks.0.9" "conv neck.deblocks.2.0"; do
  echo "== $op" >> $O
  PMX_LIB=paper_2601_12638_b200/libpmx_trace.so timeout 300 python tools/op_profile.py --op "$op" --batch 1 --trace --time 2>&1 | grep -v "per epilogue warp" | head -24 >> $O
done
