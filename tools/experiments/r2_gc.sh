#!/bin/bash
# warp-cooperative gather producer: parity + A/B (PMX_GATHER_COOP=0/1) + bench
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_gc.log
: > $O
timeout 900 python -m pytest tests/test_gpu_gather.py tests/test_gpu_forward.py tests/test_gpu_conv_tc.py -x -q 2>&1 | tail -3 >> $O
for m in 1 0 1 0; do
  for plan in "FP16: 2,18,19,20" "INT8"; do
    PMX_GATHER_COOP=$m timeout 300 python tools/op_profile.py --op "conv backbone.blocks.0.0" --plan "$plan" --time 2>&1 | grep " us" | sed "s/^/coop$m [$plan] /" >> $O
  done
done
for m in 1 0; do
  PMX_GATHER_COOP=$m timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2_gc.json 2>gpurun_out/r2_gc.err
  python - gpurun_out/r2_gc.json $m >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
L=d["latency"]
print("coop",sys.argv[2],round(d["value"]), round(d["e2e"]["value"]), d["op_ms"], "b1", round(L["mixed_b1_p50_ms"],4), "int8", round(L["int8_c2_b1_p50_ms"],4), "b8", round(L["mixed_c3_b8_ms_per_step"],4))
PY
done
