#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_fh.log
: > $O
for v in 1 0; do
  PMX_FUSE_HEADS=$v timeout 400 python bench.py --steps 10 --warmup 5 --no-cpu-baseline > gpurun_out/r2_fh_$v.json 2>gpurun_out/r2_fh_$v.err
  echo "== PMX_FUSE_HEADS=$v rc=$?" >> $O
  python - gpurun_out/r2_fh_$v.json >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
print(round(d["value"]), {k: round(v,4) for k,v in d["latency"].items() if isinstance(v,(int,float))})
PY
done
PMX_FUSE_HEADS=1 PMX_NECK_STREAM=0 timeout 600 python tools/b1_prefix.py > gpurun_out/r2_prefix_fh.log 2>&1
