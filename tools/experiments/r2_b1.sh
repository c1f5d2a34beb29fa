#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_b1.log
: > $O
timeout 900 python -m pytest tests/test_gpu_conv_tc.py tests/test_gpu_forward.py -x -q 2>&1 | tail -4 >> $O
for v in 1 0; do
  PMX_ONE_SLOT=$v timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_b1_$v.json 2>gpurun_out/r2_b1_$v.err
  echo "== PMX_ONE_SLOT=$v rc=$?" >> $O
  python - gpurun_out/r2_b1_$v.json >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
print(round(d["value"]), {k: round(v,4) for k,v in d["latency"].items() if isinstance(v,(int,float))})
PY
done
PMX_LIB=paper_2601_12638_b200/libpmx_trace.so timeout 300 python tools/b1_timeline.py > gpurun_out/r2_tl_mixed2.log 2>&1
