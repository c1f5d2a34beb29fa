#!/bin/bash
export PMX_FUSE_HEADS=1
KEEP_REP=0 bash tools/ncu_ops.sh r2m "conv neck.deblocks.2.0+heads" "conv neck.deblocks.0.0+heads"
