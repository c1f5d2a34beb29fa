#!/bin/bash
# gather producer map prefetch: parity, per-op A/B against libpmx_prev.so, bench A/B
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_mp.log
: > $O
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_forward.py -x -q 2>&1 | tail -2 >> $O
for lib in libpmx.so libpmx_prev.so libpmx.so libpmx_prev.so; do
  for plan in "FP16: 2,18,19,20" "INT8"; do
    PMX_LIB=paper_2601_12638_b200/$lib timeout 300 python tools/op_profile.py --op "conv backbone.blocks.0.0" --plan "$plan" --time 2>&1 | grep " us" | sed "s/^/$lib [$plan] /" >> $O
  done
done
bash tools/r2_ab.sh
cat gpurun_out/r2_ab.log >> $O
