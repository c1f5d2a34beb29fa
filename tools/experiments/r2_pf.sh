#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
PMX_NECK_STREAM=0 timeout 600 python tools/b1_prefix.py > gpurun_out/r2_prefix.log 2>&1
