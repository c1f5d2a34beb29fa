#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_forward.py -m gpu -q -x -k "pipelined" > gpurun_out/r3d_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r3d_tests.log
timeout 600 python bench.py --steps 30 --warmup 5 --no-latency --no-cpu-baseline > gpurun_out/r3d_b2.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-latency --no-cpu-baseline --inflight 1 > gpurun_out/r3d_b1.log 2>&1
