cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_14.txt
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_14.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/bench_14.json')); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_14.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
