cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x -k "addressing or probe or hoist or portfolio or errors" 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_41.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2,0:0:1 --reps 10 2>/dev/null | tee gpurun_out/tune_41.jsonl
for v in 2 1; do ARA_MAP_MODE=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_41_m$v.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; done
