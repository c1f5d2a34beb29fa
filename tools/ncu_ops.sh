#!/bin/bash
# ncu --set full of selected engine ops (real activations, batch 32), one report per op.
# usage: tools/ncu_ops.sh <tag> "<op1>" "<op2>" ...
set -u
TAG=$1; shift
mkdir -p gpurun_out
export PMX_NO_BUILD=1
for op in "$@"; do
  f=$(echo "$op" | tr ' ().' '___')
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o gpurun_out/${TAG}_${f} python tools/op_profile.py --op "$op" > gpurun_out/${TAG}_${f}.log 2>&1
  echo "$op rc=$?" >> gpurun_out/${TAG}_ncu_rc.txt
  python tools/ncu_summary.py gpurun_out/${TAG}_${f}.ncu-rep > gpurun_out/${TAG}_${f}_summary.txt 2>&1
  ncu -i gpurun_out/${TAG}_${f}.ncu-rep --page details --csv > gpurun_out/${TAG}_${f}_details.csv 2>&1
  ncu -i gpurun_out/${TAG}_${f}.ncu-rep --page source --csv > gpurun_out/${TAG}_${f}_source.csv 2>&1
  [ "${KEEP_REP:-0}" = 1 ] || rm -f gpurun_out/${TAG}_${f}.ncu-rep
done
