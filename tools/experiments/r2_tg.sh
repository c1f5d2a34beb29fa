#!/bin/bash
export PMX_NO_BUILD=1 PMX_LIB=$PWD/build/trace/libpmx.so
mkdir -p gpurun_out
timeout 300 python tools/op_profile.py --op "conv backbone.blocks.0.0" --trace > gpurun_out/r2_tg.log 2>&1
