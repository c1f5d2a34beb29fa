#!/bin/bash
# PFN pillars per warp at small batch: parity + batch-1 A/B (PMX_PFN_PPW=32 = before)
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_ppw.log
: > $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py tests/test_gpu_fullsize_parity.py -x -q 2>&1 | tail -2 >> $O
for m in 0 32 0 32 16; do
  echo "ppw=$m $(PMX_PFN_PPW=$m timeout 300 python tools/b1_probe.py 2>&1 | tail -1)" >> $O
done
PMX_NECK_STREAM=0 timeout 600 python tools/b1_prefix.py 2>&1 | head -5 >> $O
