cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "tiny or ragged or fuzz or headline_size" 2>&1 | tail -2
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_52.jsonl
timeout 300 python tools/tune_scan.py --config sweep-ragged --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_52.jsonl
timeout 300 python tools/tune_scan.py --config sweep-e8 --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_52.jsonl
timeout 300 python tools/tune_scan.py --config headline --precision 32 --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_52.jsonl
