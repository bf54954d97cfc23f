cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_7.txt
for cfg in headline sweep-ragged portfolio; do for sc in static dynamic; do timeout 300 python tools/tune_scan.py --config $cfg --variants 0:0 --sched $sc --reps 5; done; done | tee gpurun_out/tune_7.jsonl
