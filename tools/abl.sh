export PMX_NO_BUILD=1
for v in base abl1 abl2 abl3; do
  if [ $v = base ]; then unset PMX_LIB; else export PMX_LIB=$PWD/build/$v/libpmx.so; fi
  for op in "conv neck.deblocks.0.0" "conv neck.deblocks.2.0" "conv backbone.blocks.0.3" "conv backbone.blocks.1.3"; do
    python tools/op_profile.py --op "$op" --time 2>&1 | grep " us" | sed "s/^/$v /"
  done
done
