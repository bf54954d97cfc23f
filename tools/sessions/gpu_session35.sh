cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_35.txt
timeout 600 python bench.py --precision 32 --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_35_f32.json 2>/dev/null | cut -c1-400
timeout 300 python tools/time_metrics.py 2>&1 | tee gpurun_out/time_metrics_35.jsonl
