#!/bin/bash
# fused deconv+heads at batch 32 after the requant fallback change (PMX_FUSE_HEADS=1 forces it)
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_fh2.log
: > $O
for m in 1 0 1 0; do
  PMX_FUSE_HEADS=$m timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2_fh2.json 2>gpurun_out/r2_fh2.err
  python - gpurun_out/r2_fh2.json $m >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
L=d["latency"]; pl=d["roofline"]["per_layer_ms"]
conv_tail=sum(v for k,v in pl.items() if "deblocks" in k or "heads" in k)
print("fuse",sys.argv[2],round(d["value"]), "deconv+heads ms", round(conv_tail,4), "b1", round(L["mixed_b1_p50_ms"],4), "int8", round(L["int8_c2_b1_p50_ms"],4), "b8", round(L["mixed_c3_b8_ms_per_step"],4))
PY
done
