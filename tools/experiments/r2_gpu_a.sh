#!/bin/bash
# round-2 GPU pass: the whole -m gpu suite (full-size parity included) + one bench line
T=${1:-r2}
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=25 > gpurun_out/${T}_tests.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench.log 2>&1
echo "rc=$?" >> gpurun_out/${T}_bench.log
