#!/bin/bash
# A/B of the slot pass without atomics (PMX_SLOT_RANK=1, default) vs its own atomics (=0):
# pillarize parity tests, then alternating default bench lines on the same box
export PMX_NO_BUILD=1; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "pillar or fullsize or small_end_to_end" > gpurun_out/sr_tests.log 2>&1
echo rc=$? >> gpurun_out/sr_tests.log
for i in 1 2; do
  for v in 1 0; do
    PMX_SLOT_RANK=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/sr_${v}_${i}.log 2>&1
    python -c "
import json; d=json.loads([x for x in open('gpurun_out/sr_${v}_${i}.log') if x.startswith('{')][-1])
print('rank=$v run=$i', round(d['value']), round(d['e2e']['value']), d['op_ms']['pillarize'], d['latency']['mixed_b1_p50_ms'], d['latency']['int8_c2_b1_p50_ms'], d['latency']['mixed_c3_b8_ms_per_step'])
" >> gpurun_out/sr_summary.txt 2>&1
  done
done
