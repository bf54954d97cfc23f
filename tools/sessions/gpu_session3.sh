cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_3.txt
timeout 600 python tools/tune_scan.py --variants 4:0,4:5,4:6,2:0,2:4,2:5,1:0 | tee gpurun_out/tune_3.jsonl
