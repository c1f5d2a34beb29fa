#!/bin/bash
# Same-box A/B of two prebuilt libraries (build/ab/libpmx_old.so vs libpmx_new.so):
# parity tests selected by $1 on the new one, then alternating default bench lines
export PMX_NO_BUILD=1; mkdir -p gpurun_out
K=${1:-pillar}
cp build/ab/libpmx_new.so paper_2601_12638_b200/libpmx.so
timeout 900 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/ab_tests.log 2>&1
echo rc=$? >> gpurun_out/ab_tests.log
for i in 1 2; do
  for v in old new; do
    cp build/ab/libpmx_$v.so paper_2601_12638_b200/libpmx.so
    timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${v}_${i}.log 2>&1
    python -c "
import json; d=json.loads([x for x in open('gpurun_out/ab_${v}_${i}.log') if x.startswith('{')][-1])
print('$v run=$i', round(d['value']), round(d['e2e']['value']), d['op_ms'], d['latency']['mixed_b1_p50_ms'], d['latency']['int8_c2_b1_p50_ms'], d['latency']['mixed_c3_b8_ms_per_step'])
" >> gpurun_out/ab_summary.txt 2>&1
  done
done
cp build/ab/libpmx_new.so paper_2601_12638_b200/libpmx.so
