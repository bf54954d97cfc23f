cd $GRAFT_REPO_ROOT
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2,0:2:2,0:3:2 --reps 10 --env ARA_SCAN_DEPTH=4 2>/dev/null | tee gpurun_out/tune_50.jsonl
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2,4:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_50.jsonl
