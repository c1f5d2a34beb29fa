#!/bin/bash
# decode anchors-per-CTA at batch 1 (PMX_DECODE_CHUNK) after the rank-sort finish
export PMX_NO_BUILD=1
mkdir -p gpurun_out
O=gpurun_out/r2_dch.log
: > $O
for c in 0 2048 1024 0 2048 1024 8192; do
  echo "chunk=$c $(PMX_DECODE_CHUNK=$c timeout 300 python tools/b1_probe.py 2>&1 | tail -1)" >> $O
done
