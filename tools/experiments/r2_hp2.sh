#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_conv_tc.py -x -q 2>&1 | tail -15 > gpurun_out/r2_hp2.log
