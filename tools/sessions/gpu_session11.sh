cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -s 2>&1 | grep -E "passed|failed|fp32 vs|Error|error" | tail -8 | tee gpurun_out/pytest_gpu_11.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0 --reps 5 | tee gpurun_out/tune_11.jsonl
