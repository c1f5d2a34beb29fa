#!/bin/bash
# batch-8 (config 3) knobs: PFN pillars per warp, decode anchors per CTA
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_b8.log
: > $O
for cfg in "X=0" "PMX_PFN_PPW=16" "PMX_PFN_PPW=8" "PMX_DECODE_CHUNK=8192" "PMX_DECODE_CHUNK=4096" "X=0"; do
  env $cfg timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2_b8.json 2>gpurun_out/r2_b8.err
  python - gpurun_out/r2_b8.json "$cfg" >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
L=d["latency"]
print(sys.argv[2], round(d["value"]), d["op_ms"]["pfn"], d["op_ms"]["decode"], "b1", round(L["mixed_b1_p50_ms"],4), "int8", round(L["int8_c2_b1_p50_ms"],4), "b8", round(L["mixed_c3_b8_ms_per_step"],4))
PY
done
