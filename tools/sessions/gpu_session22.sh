cd $GRAFT_REPO_ROOT
for m in 1 2; do
ARA_MAP_MODE=$m timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_22_m$m python tools/tune_scan.py --config headline --variants 0:0:$m --reps 1 > gpurun_out/ncu_22_m$m.log 2>&1
ncu -i gpurun_out/prof_scan_22_m$m.ncu-rep --page raw --csv > gpurun_out/prof_scan_22_m${m}_raw.csv 2>&1
done
ls -la gpurun_out | tail
