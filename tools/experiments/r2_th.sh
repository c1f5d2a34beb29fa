#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_th.log
: > $O
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_forward.py -x -q 2>&1 | tail -3 >> $O
timeout 300 python tools/decode_probe.py --batch 1 >> $O 2>&1
timeout 300 python tools/decode_probe.py --batch 32 >> $O 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_th.json 2>gpurun_out/r2_th.err
python - gpurun_out/r2_th.json >> $O <<'PY'
import json,sys
d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
print(round(d["value"]), d["op_ms"], {k: round(v,4) for k,v in d["latency"].items() if isinstance(v,(int,float))})
PY
