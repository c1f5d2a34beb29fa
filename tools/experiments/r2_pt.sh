#!/bin/bash
export PMX_NO_BUILD=1 PMX_LIB=$PWD/build/ptrace/libpmx.so
mkdir -p gpurun_out
timeout 300 python tools/b1_ops.py 2>&1 | grep "pfn trace" | tail -24 > gpurun_out/r2_pt.log
