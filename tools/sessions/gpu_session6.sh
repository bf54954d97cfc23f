cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_6.txt
for sc in static dynamic; do timeout 300 python tools/tune_scan.py --variants 0:0 --sched $sc --reps 5; done | tee gpurun_out/tune_6h.jsonl
for sc in static dynamic; do timeout 300 python tools/tune_scan.py --config sweep-ragged --variants 0:0 --sched $sc --reps 5; done | tee gpurun_out/tune_6r.jsonl
for c in sweep-e4 sweep-e8 sweep-e32 sweep-e64 sweep-k500 sweep-k2000; do timeout 300 python tools/tune_scan.py --config $c --variants 0:0 --reps 3; done | tee gpurun_out/tune_6s.jsonl
