#!/bin/bash
# split-graph streaming: pipelined tests, then e2e A/B (PMX_PIPE_SPLIT=0/1)
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_sp.log
: > $O
timeout 900 python -m pytest tests/test_gpu_forward.py -x -q -k "pipelined" 2>&1 | tail -3 >> $O
for m in 1 0 1 0; do
  PMX_PIPE_SPLIT=$m timeout 400 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-latency > gpurun_out/r2_sp.json 2>gpurun_out/r2_sp.err
  python - gpurun_out/r2_sp.json $m >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
print("split",sys.argv[2],round(d["value"]), "e2e", round(d["e2e"]["value"]), d["e2e"]["ms_per_step"])
PY
done
