#!/bin/bash
# same-box A/B of the current library against libpmx_prev.so (bench latency + per-op)
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_ab.log
: > $O
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py tests/test_gpu_gather.py -x -q 2>&1 | tail -2 >> $O
for lib in libpmx.so libpmx_prev.so libpmx.so libpmx_prev.so; do
  PMX_LIB=paper_2601_12638_b200/$lib timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_ab.json 2>gpurun_out/r2_ab.err
  echo "== $lib rc=$?" >> $O
  python - gpurun_out/r2_ab.json >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
L=d["latency"]
print(round(d["value"]), d["op_ms"]["pillarize"], d["op_ms"]["decode"], "b1 mixed", round(L["mixed_b1_p50_ms"],4), "int8", round(L["int8_c2_b1_p50_ms"],4), "b8", round(L["mixed_c3_b8_ms_per_step"],4))
PY
done
