# Session 74: ncu of the F4 kernel with per-event increments (what the 4.4 ms over max-only is).
cd $GRAFT_REPO_ROOT
timeout 1500 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section Occupancy --section LaunchStats --clock-control none -k regex:scan_kernel --launch-skip 14 --launch-count 1 -o gpurun_out/prof_f4inc_74 python tools/time_f4.py > gpurun_out/ncu_f4inc_74.log 2>&1; tail -3 gpurun_out/ncu_f4inc_74.log
timeout 300 ncu -i gpurun_out/prof_f4inc_74.ncu-rep --page details --csv > gpurun_out/f4inc_74_details.csv 2>&1; wc -l gpurun_out/f4inc_74_details.csv
