cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_23.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:1,0:2:1,0:0:2,0:2:2,0:0:0,0:2:0 --reps 5 --flags 4 2>&1 | tee gpurun_out/tune_23.jsonl
