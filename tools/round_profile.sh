#!/bin/bash
# Round-end evidence on the GPU box: default bench line, ncu launch list of the same
# command, per-kernel DRAM traffic of one step, one --set full capture of the top conv.
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
export PMX_NO_BUILD=1
timeout 900 python bench.py > $OUT/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> $OUT/${TAG}_bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-latency --no-cpu-baseline > $OUT/${TAG}_ncu_list.log 2>&1
echo "list rc=$?" >> $OUT/${TAG}_ncu_list.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  --profile-from-start off --csv python tools/op_profile.py --op all > $OUT/${TAG}_traffic.csv 2> $OUT/${TAG}_traffic.err
for op in "conv neck.deblocks.0.0" "conv backbone.blocks.0.0" "conv backbone.blocks.2.3" "conv backbone.blocks.1.3" "pfn"; do
  f=$(echo "$op" | tr ' ().' '___')
  timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off \
    -o $OUT/${TAG}_${f} python tools/op_profile.py --op "$op" > $OUT/${TAG}_${f}.log 2>&1
  python tools/ncu_summary.py $OUT/${TAG}_${f}.ncu-rep > $OUT/${TAG}_${f}_summary.txt 2>&1
  rm -f $OUT/${TAG}_${f}.ncu-rep
done
