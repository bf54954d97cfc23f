cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_38.txt
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2,0:0:1 --reps 10 2>/dev/null | tee gpurun_out/tune_38.jsonl
timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_38.jsonl
for c in sweep-e8 sweep-e32 sweep-e64 sweep-ragged; do timeout 300 python tools/tune_scan.py --config $c --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_38.jsonl; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_38 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
