#!/bin/bash
T=${1:-r2}
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --no-latency --no-cpu-baseline > gpurun_out/${T}_base.log 2>&1
PMX_HSWZ_W=10 timeout 600 python bench.py --steps 20 --warmup 5 --no-latency --no-cpu-baseline > gpurun_out/${T}_w10.log 2>&1
PMX_HALO_SWZ=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-latency --no-cpu-baseline > gpurun_out/${T}_noswz.log 2>&1
PMX_ESTAGE=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-latency --no-cpu-baseline > gpurun_out/${T}_noestage.log 2>&1
