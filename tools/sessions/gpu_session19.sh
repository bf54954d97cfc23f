cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_19.txt
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_19.json 2> gpurun_out/bench_19.err
timeout 900 python bench.py --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_19_portfolio.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_19.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_19 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:portfolio_kernel -s 1 -c 1 -o gpurun_out/prof_portfolio_19 python tools/tune_scan.py --config portfolio --variants 0:0 --reps 1 > /dev/null 2>&1
ls gpurun_out | tail -12
