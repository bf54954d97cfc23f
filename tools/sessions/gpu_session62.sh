cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_62.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_62.json 2> gpurun_out/bench_62.err | cut -c1-100
timeout 900 python bench.py --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_62_portfolio.json 2>/dev/null | cut -c1-100
timeout 900 python bench.py --hoist --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_62_hoist.json 2>/dev/null | cut -c1-100
timeout 900 python bench.py --hoist --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_62_hoist_portfolio.json 2>/dev/null | cut -c1-100
timeout 600 python bench.py --config sweep-ragged --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_62_ragged.json 2>/dev/null | cut -c1-100
timeout 600 python bench.py --precision 32 --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_62_f32.json 2>/dev/null | cut -c1-100
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_62.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > gpurun_out/sanitizer_racecheck_62.txt 2>&1; tail -1 gpurun_out/sanitizer_racecheck_62.txt
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_cases.py > gpurun_out/sanitizer_memcheck_62.txt 2>&1; tail -1 gpurun_out/sanitizer_memcheck_62.txt
timeout 300 python tools/time_metrics.py 2>&1 | tee gpurun_out/time_metrics_62.jsonl > /dev/null
timeout 300 python tools/time_metrics_rows.py 2>&1 | tee gpurun_out/time_metrics_rows_62.jsonl > /dev/null
