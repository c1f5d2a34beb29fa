export PMX_NO_BUILD=1
for eg in 2 4 1; do
  for op in "conv neck.deblocks.0.0" "conv neck.deblocks.1.0" "conv neck.deblocks.2.0" "conv backbone.blocks.1.3" "conv backbone.blocks.0.3" "conv heads(fused)"; do
    PMX_EGROUPS=$eg python tools/op_profile.py --op "$op" --time 2>&1 | grep " us" | sed "s/^/eg=$eg /"
  done
done
