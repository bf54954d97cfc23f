cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_2.txt
timeout 600 python tools/tune_scan.py --variants 4:0,4:3,4:4,2:0,2:3,1:0 | tee gpurun_out/tune_2.jsonl
ARA_SCAN_GROUP=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_g2 python tools/tune_scan.py --variants 2:0 --reps 1 > gpurun_out/ncu_2.log 2>&1
tail -2 gpurun_out/ncu_2.log
