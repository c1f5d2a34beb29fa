#!/bin/bash
export PMX_NO_BUILD=1
bash tools/ncu_ops.sh r2t "conv neck.deblocks.0.0" "conv neck.deblocks.1.0" "pillarize" "pfn"
