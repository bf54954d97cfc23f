cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_26.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:0,0:0:1,0:0:2 --reps 5 2>&1 | tee gpurun_out/tune_26.jsonl
