#!/bin/bash
# Quick GPU iteration: conv parity tests + a short bench line (per-layer ms).
# usage: tools/quick_gpu.sh <tag> [pytest -k expr]
TAG=${1:-q}
K=${2:-conv}
mkdir -p gpurun_out
export PMX_NO_BUILD=1
timeout 600 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-latency --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
