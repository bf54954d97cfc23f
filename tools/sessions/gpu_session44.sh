cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x -k "f32" 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_44.txt
timeout 600 python bench.py --precision 32 --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_44_f32.json 2>/dev/null | cut -c1-200
for c in sweep-e8 sweep-e32 sweep-e64; do timeout 300 python tools/tune_scan.py --config $c --precision 32 --variants 0:0:2 --reps 3 2>/dev/null | tee -a gpurun_out/tune_44.jsonl; done
