#!/bin/bash
export PMX_NO_BUILD=1
export PMX_LIB=$PWD/build/trace/libpmx.so
mkdir -p gpurun_out
O=gpurun_out/r2_tr.log
: > $O
for m in 0 1; do
  for op in "conv neck.deblocks.0.0" "conv neck.deblocks.2.0"; do
    echo "== res$m $op" >> $O
    PMX_GEMM_RES=$m timeout 300 python tools/op_profile.py --op "$op" --trace >> $O 2>&1
  done
done
