#!/bin/bash
# batch-1 breakdown: in-graph per-op increments + ncu launch list of one b1 graph
export PMX_NO_BUILD=1 PMX_GEMM_RES=0
mkdir -p gpurun_out
PMX_NECK_STREAM=0 timeout 600 python tools/b1_prefix.py > gpurun_out/r2_b1x_prefix.log 2>&1
timeout 300 python tools/b1_probe.py > gpurun_out/r2_b1x_probe.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_b1x_launches.csv \
  python tools/b1_ops.py > gpurun_out/r2_b1x_ops.log 2>&1
