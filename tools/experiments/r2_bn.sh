#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_bn.log
: > $O
for bn in 256 64 128 32; do
  for op in "conv neck.deblocks.0.0" "conv neck.deblocks.1.0" "conv neck.deblocks.2.0"; do
    PMX_DECONV_BN=$bn timeout 300 python tools/op_profile.py --op "$op" --time 2>&1 | grep " us" | sed "s/^/bn$bn /" >> $O
  done
done
