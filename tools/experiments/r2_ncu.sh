#!/bin/bash
KEEP_REP=0 bash tools/ncu_ops.sh r2s "pfn" "pillarize"
