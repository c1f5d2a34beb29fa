#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qat.py -q -s -x 2>&1 | tail -40 > gpurun_out/r2_qat.log
