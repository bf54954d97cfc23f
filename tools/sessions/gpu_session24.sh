cd $GRAFT_REPO_ROOT
ARA_MAP_MODE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_24_m1 python tools/tune_scan.py --config headline --variants 0:0:1 --reps 1 > gpurun_out/ncu_24.log 2>&1
ncu -i gpurun_out/prof_scan_24_m1.ncu-rep --page raw --csv > gpurun_out/prof_scan_24_m1_raw.csv 2>&1
ncu -i gpurun_out/prof_scan_24_m1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_scan_24_m1_sass.csv 2>&1
ls -la gpurun_out | tail -4
