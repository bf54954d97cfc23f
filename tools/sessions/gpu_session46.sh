cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_46.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2 --reps 10 2>/dev/null | tee gpurun_out/tune_46.jsonl
timeout 300 python tools/tune_scan.py --config sweep-ragged --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_46.jsonl
timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_46.jsonl
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_46.json 2> gpurun_out/bench_46.err | cut -c1-200
timeout 900 python bench.py --hoist --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_46_hoist.json 2>/dev/null | cut -c1-200
timeout 600 python bench.py --config sweep-ragged --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_46_ragged.json 2>/dev/null | cut -c1-200
