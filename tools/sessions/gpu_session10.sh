cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_10.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0 --reps 5 | tee gpurun_out/tune_10.jsonl
