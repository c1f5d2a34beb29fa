#!/bin/bash
# CTA-pair (cta_group::2) conv: parity tests, then A/B bench (PMX_PAIR=0 vs default)
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_pair.log
: > $O
timeout 900 python -m pytest tests/test_gpu_conv_tc.py -x -q  2>&1 | tail -15 >> $O
for v in 0 1; do
  PMX_PAIR=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-latency > gpurun_out/r2_pair_b$v.json 2>gpurun_out/r2_pair_b$v.err
  echo "== PMX_PAIR=$v rc=$?" >> $O
  python tools/show_bench.py gpurun_out/r2_pair_b$v.json | head -1 >> $O 2>&1
done
