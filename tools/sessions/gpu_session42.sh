cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_42.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2,0:0:1 --reps 10 2>/dev/null | tee gpurun_out/tune_42.jsonl
timeout 300 python tools/tune_scan.py --config sweep-h10 --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_42.jsonl
timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2,0:0:1 --reps 5 2>/dev/null | tee -a gpurun_out/tune_42.jsonl
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_42.json 2> gpurun_out/bench_42.err | cut -c1-250
timeout 900 python bench.py --hoist --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_42_hoist.json 2>/dev/null | cut -c1-250
