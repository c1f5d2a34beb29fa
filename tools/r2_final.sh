#!/bin/bash
# round-2 evidence: GPU tests + smoke, then tools/round_profile.sh (bench line, ncu launch
# list, per-kernel traffic, --set full captures), the reference arm, and the sweep
set -u
TAG=${1:-r2x}
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1
bash tools/round_profile.sh $TAG
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.log 2>&1
