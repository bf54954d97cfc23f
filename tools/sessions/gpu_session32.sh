cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_32.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke_32.txt
for lib in "" imax; do
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2,0:0:1 --reps 10 2>/dev/null | tee -a gpurun_out/tune_32.jsonl
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:1 --reps 3 2>/dev/null | tee -a gpurun_out/tune_32.jsonl
done
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_32.json 2> gpurun_out/bench_32.err
timeout 900 python bench.py --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_32_portfolio.json 2>/dev/null
timeout 600 python bench.py --config sweep-ragged --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_32_ragged.json 2>/dev/null
timeout 600 python bench.py --precision 32 --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_32_f32.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_32_ref.json 2> gpurun_out/bench_32_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_32.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | tail -12
