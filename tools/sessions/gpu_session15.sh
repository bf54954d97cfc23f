cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x --durations=8 2>&1 | tail -14 | tee gpurun_out/pytest_gpu_15.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_15.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
