cd $GRAFT_REPO_ROOT
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:1,0:0:2,0:0:0,4:0:1 --reps 5 2>&1 | tee gpurun_out/tune_28.jsonl
timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:1,0:0:2,0:0:0 --reps 3 2>&1 | tee -a gpurun_out/tune_28.jsonl
timeout 300 python tools/tune_scan.py --config sweep-h10 --variants 0:0:2,0:0:0 --reps 3 2>&1 | tee -a gpurun_out/tune_28.jsonl
