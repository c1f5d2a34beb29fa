#!/bin/bash
# quant16_sel (per-value fixup of flagged values): parity + per-op A/B vs libpmx_prev.so + bench A/B
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_qs.log
: > $O
timeout 1200 python -m pytest tests/test_gpu_conv_tc.py tests/test_gpu_forward.py tests/test_gpu_kernels.py tests/test_gpu_fullsize_parity.py -x -q 2>&1 | tail -2 >> $O
for lib in libpmx.so libpmx_prev.so libpmx.so libpmx_prev.so; do
  for op in "conv neck.deblocks.0.0" "conv backbone.blocks.0.9" "conv backbone.blocks.1.15"; do
    PMX_LIB=paper_2601_12638_b200/$lib timeout 300 python tools/op_profile.py --op "$op" --time 2>&1 | grep " us" | sed "s/^/$lib /" >> $O
  done
done
bash tools/r2_ab.sh
cat gpurun_out/r2_ab.log >> $O
