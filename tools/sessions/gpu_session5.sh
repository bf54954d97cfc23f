cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_5.txt
timeout 600 python tools/tune_scan.py --variants 2:0,4:0 | tee gpurun_out/tune_5.jsonl
timeout 600 python tools/tune_scan.py --config portfolio --variants 2:0,4:0 --reps 5 | tee gpurun_out/tune_5p.jsonl
timeout 900 python bench.py --config portfolio --steps 5 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_5p.json 2> gpurun_out/bench_5p.err
