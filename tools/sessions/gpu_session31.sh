cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tee gpurun_out/gpu_31.txt
cat MEASURED_PEAKS.json 2>/dev/null | tee gpurun_out/measured_peaks_31.json
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_31.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke_31.txt
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_31.json 2> gpurun_out/bench_31.err
timeout 900 python bench.py --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_31_portfolio.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_31.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_31 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:portfolio_kernel -s 1 -c 1 -o gpurun_out/prof_portfolio_31 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 1 > /dev/null 2>&1
ls gpurun_out | tail -12
