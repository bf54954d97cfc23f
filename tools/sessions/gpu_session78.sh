# Session 78: ncu --set full with source of the final headline scan launch (hot-loop stall map).
cd $GRAFT_REPO_ROOT
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:scan_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/prof_scan_78 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_scan_78.log 2>&1; tail -2 gpurun_out/ncu_scan_78.log
