cd $GRAFT_REPO_ROOT
for m in 2 1 0; do ARA_MAP_MODE=$m timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | sed "s/^/mode $m: /"; done | tee gpurun_out/pytest_gpu_21.txt
for c in headline sweep-h10 portfolio sweep-e64; do timeout 300 python tools/tune_scan.py --config $c --variants 0:0:0,0:0:1,0:0:2 --reps 5 --flags 4; done 2>&1 | tee gpurun_out/tune_21.jsonl
