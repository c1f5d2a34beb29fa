#!/bin/bash
# source-level ncu captures of the main conv kernels; the SASS source page (with stall
# samples / executed instructions) is exported as csv on the box, the reports dropped
export PMX_NO_BUILD=1
mkdir -p gpurun_out
for op in "conv backbone.blocks.0.0" "conv backbone.blocks.0.3" "conv backbone.blocks.1.3" "conv backbone.blocks.2.3" "conv heads(fused)"; do
  f=$(echo "$op" | tr ' ().' '___')
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o /tmp/src_${f} python tools/op_profile.py --op "$op" > gpurun_out/src_${f}.log 2>&1
  ncu -i /tmp/src_${f}.ncu-rep --page source --csv --print-source sass > /tmp/src_${f}.csv 2>&1
  gzip -c /tmp/src_${f}.csv > gpurun_out/src_${f}.csv.gz
done
