#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3i_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3i_tests.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r3i_bench.log 2>&1
