#!/bin/bash
T=${1:-r2}
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py tests/test_gpu_fullsize_parity.py -m gpu -q -x > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-latency --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1
