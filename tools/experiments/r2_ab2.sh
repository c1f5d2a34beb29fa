#!/bin/bash
# same-box A/B of the batch-32 step: current library vs libpmx_prev.so (per-layer ms)
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_ab2.log
: > $O
timeout 1200 python -m pytest tests/test_gpu_conv_tc.py tests/test_gpu_forward.py -x -q 2>&1 | tail -2 >> $O
for lib in libpmx.so libpmx_prev.so libpmx.so libpmx_prev.so; do
  PMX_LIB=paper_2601_12638_b200/$lib timeout 400 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-latency > gpurun_out/r2_ab2_$lib.json 2>gpurun_out/r2_ab2.err
  echo "== $lib rc=$?" >> $O
  python - gpurun_out/r2_ab2_$lib.json >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
pl=d["roofline"]["per_layer_ms"]
print(round(d["value"]), "conv", d["op_ms"]["conv"], " ".join(f"{k.split()[-1].replace('backbone.blocks.','b').replace('neck.deblocks.','d')}={v:.4f}" for k,v in pl.items()))
PY
done
