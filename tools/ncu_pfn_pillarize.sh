export PMX_NO_BUILD=1
ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:pfn_points -o gpurun_out/s3_pfn python tools/op_profile.py --op pfn > gpurun_out/s3_pfn.log 2>&1
python tools/ncu_summary.py gpurun_out/s3_pfn.ncu-rep > gpurun_out/s3_pfn_summary.txt 2>&1
ncu -i gpurun_out/s3_pfn.ncu-rep --page source --csv > gpurun_out/s3_pfn_source.csv 2>&1
ncu -i gpurun_out/s3_pfn.ncu-rep --page details --csv > gpurun_out/s3_pfn_details.csv 2>&1
ncu --set full --clock-control none --profile-from-start off -k regex:"emit|bin_kernel|slot_kernel" -o gpurun_out/s3_pil python tools/op_profile.py --op pillarize > gpurun_out/s3_pil.log 2>&1
python tools/ncu_summary.py gpurun_out/s3_pil.ncu-rep > gpurun_out/s3_pil_summary.txt 2>&1
rm -f gpurun_out/*.ncu-rep
