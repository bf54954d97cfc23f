cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv | tee gpurun_out/gpu_43.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/smoke_43.txt
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_43.json 2> gpurun_out/bench_43.err | cut -c1-200
timeout 900 python bench.py --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_43_portfolio.json 2>/dev/null | cut -c1-200
timeout 600 python bench.py --config sweep-ragged --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_43_ragged.json 2>/dev/null | cut -c1-200
timeout 600 python bench.py --precision 32 --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_43_f32.json 2>/dev/null | cut -c1-200
timeout 900 python bench.py --hoist --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_43_hoist.json 2>/dev/null | cut -c1-200
timeout 900 python bench.py --hoist --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_43_hoist_portfolio.json 2>/dev/null | cut -c1-200
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_43_ref.json 2> gpurun_out/bench_43_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_43.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_43 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:portfolio_kernel -s 1 -c 1 -o gpurun_out/prof_portfolio_43 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 1 > /dev/null 2>&1
bash tools/sweep.sh gpurun_out/sweep_43.jsonl
ls gpurun_out | grep _43
