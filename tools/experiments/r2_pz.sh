#!/bin/bash
# persistent pillarize + rank-sort decode: parity, then batch-1 / batch-8 A/B
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_pz.log
: > $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py tests/test_gpu_decode_nms.py -x -q 2>&1 | tail -5 >> $O
for m in 1 0 1 0; do
  echo "persist=$m $(PMX_PILLARIZE_PERSIST=$m timeout 300 python tools/b1_probe.py 2>&1 | tail -1)" >> $O
done
PMX_NECK_STREAM=0 timeout 600 python tools/b1_prefix.py 2>&1 | tail -25 >> $O
