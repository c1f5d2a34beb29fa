export PMX_NO_BUILD=1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:pfn_points -o gpurun_out/s5_pfn python tools/op_profile.py --op pfn > gpurun_out/s5_pfn.log 2>&1
ncu -i gpurun_out/s5_pfn.ncu-rep --page source --csv > gpurun_out/s5_pfn_source.csv 2>&1
python tools/ncu_summary.py gpurun_out/s5_pfn.ncu-rep > gpurun_out/s5_pfn_summary.txt 2>&1
rm -f gpurun_out/s5_pfn.ncu-rep
