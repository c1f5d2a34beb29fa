#!/bin/bash
# deconv epilogue study: ablation timings (base / abl1 no compute+store / abl2 no global
# store / abl3 raw store) and one --set full capture with source counters kept
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_dc.log
: > $O
for v in base abl1 abl2 abl3; do
  if [ $v = base ]; then unset PMX_LIB; else export PMX_LIB=$PWD/build/$v/libpmx.so; fi
  for op in "conv neck.deblocks.0.0" "conv neck.deblocks.1.0" "conv neck.deblocks.2.0"; do
    timeout 300 python tools/op_profile.py --op "$op" --time 2>&1 | grep " us" | sed "s/^/$v /" >> $O
  done
done
unset PMX_LIB
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -o gpurun_out/r2_dc0 python tools/op_profile.py --op "conv neck.deblocks.0.0" > gpurun_out/r2_dc0.log 2>&1
