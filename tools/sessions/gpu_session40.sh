cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_40.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2,0:0:1 --reps 10 2>/dev/null | tee gpurun_out/tune_40.jsonl
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2 --reps 10 --env ARA_MAP_PROBE=0 2>/dev/null | tee -a gpurun_out/tune_40.jsonl
timeout 300 python tools/tune_scan.py --config sweep-h10 --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_40.jsonl
timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_40.jsonl
for c in sweep-e8 sweep-e32; do timeout 300 python tools/tune_scan.py --config $c --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_40.jsonl; done
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_40.json 2> gpurun_out/bench_40.err | cut -c1-250
timeout 900 python bench.py --hoist --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_40_hoist.json 2>/dev/null | cut -c1-250
