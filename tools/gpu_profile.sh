#!/bin/bash
# Run on the GPU box: plain bench line, then the ncu launch list and one full capture of the top kernel.
# usage: tools/gpu_profile.sh <tag>
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
export PMX_NO_BUILD=1
CMD="python bench.py --steps 2 --warmup 3 --no-latency --no-cpu-baseline"
$CMD > $OUT/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_ncu_list.log 2>&1
echo "list rc=$?" >> $OUT/${TAG}_ncu_list.log
$CMD > $OUT/${TAG}_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 40 -c 4 -o $OUT/${TAG}_conv_tc $CMD > $OUT/${TAG}_ncu_full.log 2>&1
echo "full rc=$?" >> $OUT/${TAG}_ncu_full.log
