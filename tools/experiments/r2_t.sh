#!/bin/bash
export PMX_NO_BUILD=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2_t.log 2>&1; echo "rc=$?" >> gpurun_out/r2_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" >> gpurun_out/r2_t.log 2>&1
