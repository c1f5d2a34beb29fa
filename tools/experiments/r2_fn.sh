#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_fn.log
: > $O
timeout 900 python -m pytest tests/test_gpu_heads_fusion.py tests/test_gpu_forward.py tests/test_gpu_fullsize_parity.py -x -q 2>&1 | tail -3 >> $O
for v in 1 0; do
  PMX_NECK_STREAM=$v timeout 400 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2_fn_$v.json 2>gpurun_out/r2_fn_$v.err
  echo "== PMX_NECK_STREAM=$v rc=$?" >> $O
  python - gpurun_out/r2_fn_$v.json >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
print(round(d["value"]), {k: round(v,4) for k,v in d["latency"].items() if isinstance(v,(int,float))})
PY
done
