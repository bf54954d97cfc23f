cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -k "hoist" 2>&1 | tail -15 | tee gpurun_out/pytest_gpu_36_hoist.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_36.txt
timeout 900 python bench.py --hoist --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_36_hoist.json 2>/dev/null | cut -c1-300
timeout 900 python bench.py --hoist --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_36_hoist_portfolio.json 2>/dev/null | cut -c1-300
timeout 900 python bench.py --hoist --config sweep-h10 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_36_hoist_h10.json 2>/dev/null | cut -c1-300
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hoisted_scan_kernel -s 3 -c 1 -o gpurun_out/prof_hoist_36 python bench.py --hoist --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hoisted_scan_kernel -s 3 -c 1 -o gpurun_out/prof_hoist_pf_36 python bench.py --hoist --config portfolio --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_36_hoist.csv python bench.py --hoist --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | tail -8
