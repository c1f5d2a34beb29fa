#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_dec2.log
: > $O
for b in 1 32; do timeout 300 python tools/op_profile.py --op decode --batch $b --time 2>&1 | tail -1 >> $O; done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py tests/test_gpu_decode_nms.py -x -q 2>&1 | tail -2 >> $O
PMX_NECK_STREAM=0 timeout 600 python tools/b1_prefix.py > gpurun_out/r2_prefix3.log 2>&1
tail -3 gpurun_out/r2_prefix3.log >> $O
