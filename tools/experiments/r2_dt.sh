#!/bin/bash
export PMX_NO_BUILD=1 PMX_LIB=$PWD/build/dtrace/libpmx.so
mkdir -p gpurun_out
timeout 300 python tools/b1_ops.py 2>&1 | grep "decode trace" | tail -8 > gpurun_out/r2_dt.log
