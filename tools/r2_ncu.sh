#!/bin/bash
KEEP_REP=0 bash tools/ncu_ops.sh r2q "conv backbone.blocks.1.3" "conv backbone.blocks.2.3" "conv backbone.blocks.0.3"
