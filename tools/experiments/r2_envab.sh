#!/bin/bash
# Same-box A/B of an env knob: $1 = variable, $2.. = values; parity tests (-k $TESTK) on
# the first value, then alternating default bench lines (two rounds)
export PMX_NO_BUILD=1; mkdir -p gpurun_out
VAR=$1; shift
env $VAR=$1 timeout 900 python -m pytest tests -m gpu -q -x -k "${TESTK:-pillar}" > gpurun_out/ev_tests.log 2>&1
echo rc=$? >> gpurun_out/ev_tests.log
for i in 1 2; do
  for v in "$@"; do
    env $VAR=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ev_${v}_${i}.log 2>&1
    python -c "
import json; d=json.loads([x for x in open('gpurun_out/ev_${v}_${i}.log') if x.startswith('{')][-1])
print('$VAR=$v run=$i', round(d['value']), round(d['e2e']['value']), d['op_ms'], d['latency']['mixed_b1_p50_ms'], d['latency']['int8_c2_b1_p50_ms'], d['latency']['mixed_c3_b8_ms_per_step'])
" >> gpurun_out/ev_summary.txt 2>&1
  done
done
