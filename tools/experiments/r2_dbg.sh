export PMX_NO_BUILD=1
mkdir -p gpurun_out
for e in "3 none" "3 cnt4"; do
  echo "== $e" >> gpurun_out/r2h_dbg.log
  PMX_LIB=paper_2601_12638_b200/libpmx_dbg.so timeout 120 python tools/dbg_pfn.py $e 2>&1 | grep -v "^  File\|^    \|Search for\|CUDA kernel errors\|For debugging\|Compile with" >> gpurun_out/r2h_dbg.log
done
