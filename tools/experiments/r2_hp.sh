#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_hp.log
: > $O
timeout 900 python -m pytest tests/test_gpu_conv_tc.py -x -q 2>&1 | tail -15 >> $O
timeout 900 python -m pytest tests/test_gpu_fullsize_parity.py tests/test_gpu_forward.py -x -q 2>&1 | tail -3 >> $O
for v in 1 0; do
  PMX_PAIR=$v timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-latency > gpurun_out/r2_hp_$v.json 2>gpurun_out/r2_hp_$v.err
  echo "== PMX_PAIR=$v rc=$?" >> $O
  python tools/show_bench.py gpurun_out/r2_hp_$v.json >> $O 2>&1
done
