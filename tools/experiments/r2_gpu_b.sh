#!/bin/bash
T=${1:-r2}
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tf32x3.py tests/test_gpu_heads_fusion.py -m gpu -q -s > gpurun_out/${T}_new.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_new.log
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_bench.log
