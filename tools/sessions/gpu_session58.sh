cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_58.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_58.json 2> gpurun_out/bench_58.err | cut -c1-120
timeout 900 python bench.py --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_58_portfolio.json 2>/dev/null | cut -c1-120
timeout 900 python bench.py --hoist --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_58_hoist.json 2>/dev/null | cut -c1-120
timeout 900 python bench.py --hoist --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_58_hoist_portfolio.json 2>/dev/null | cut -c1-120
timeout 600 python bench.py --hoist --config sweep-h10 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_58_hoist_h10.json 2>/dev/null | cut -c1-120
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_58_hoist.csv python bench.py --hoist --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hoisted_scan_kernel -s 3 -c 1 -o gpurun_out/prof_hoist_58 python bench.py --hoist --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
