#!/bin/bash
# GEMM resident-weight mode: parity + per-op A/B (PMX_GEMM_RES=0/1/2) + bench A/B
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_gr.log
: > $O
timeout 900 python -m pytest tests/test_gpu_conv_tc.py tests/test_gpu_forward.py tests/test_gpu_heads_fusion.py -x -q 2>&1 | tail -3 >> $O
for m in 0 1 2; do
  for op in "conv neck.deblocks.0.0" "conv neck.deblocks.1.0" "conv neck.deblocks.2.0" "conv heads(fused)"; do
    PMX_GEMM_RES=$m timeout 300 python tools/op_profile.py --op "$op" --time 2>&1 | grep " us" | sed "s/^/res$m /" >> $O
  done
done
for m in 0 1 0 1; do
  PMX_GEMM_RES=$m timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2_gr.json 2>gpurun_out/r2_gr.err
  python - gpurun_out/r2_gr.json $m >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
L=d["latency"]
print("res",sys.argv[2],round(d["value"]), round(d["e2e"]["value"]), d["op_ms"], "b1", round(L["mixed_b1_p50_ms"],4), "int8", round(L["int8_c2_b1_p50_ms"],4), "b8", round(L["mixed_c3_b8_ms_per_step"],4))
PY
done
