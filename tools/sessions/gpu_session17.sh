cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_17.txt
for pf in 1 0; do timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0 --reps 5 --env ARA_PORTFOLIO=$pf; done | tee gpurun_out/tune_17.jsonl
