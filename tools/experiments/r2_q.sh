#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_q.log
: > $O
timeout 1200 python -m pytest tests/test_gpu_conv_tc.py tests/test_gpu_fullsize_parity.py tests/test_gpu_forward.py tests/test_gpu_kernels.py -x -q 2>&1 | tail -4 >> $O
for i in 1 2; do
  timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-latency > gpurun_out/r2_q_$i.json 2>gpurun_out/r2_q_$i.err
  python tools/show_bench.py gpurun_out/r2_q_$i.json >> $O 2>&1
done
