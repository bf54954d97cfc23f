cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_29.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:1,0:0:2,0:0:0 --reps 5 2>&1 | tee gpurun_out/tune_29.jsonl
timeout 300 python tools/tune_scan.py --config sweep-h10 --variants 0:0:2,0:0:0 --reps 3 2>&1 | tee -a gpurun_out/tune_29.jsonl
timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:1,0:0:2,0:0:0 --reps 3 2>&1 | tee -a gpurun_out/tune_29.jsonl
