cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 1 -c 1 -o gpurun_out/prof_scan_portfolio python tools/tune_scan.py --config portfolio --variants 0:0 --reps 1 > /dev/null 2>&1
ls -la gpurun_out/
