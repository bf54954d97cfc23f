cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "elts_per_layer_widths or fuzz" 2>&1 | tail -2
for c in sweep-e32 sweep-e64; do for t in 1 0; do timeout 300 python tools/tune_scan.py --config $c --variants 0:0:2 --reps 5 --env ARA_SCAN_TS=$t 2>/dev/null | tee -a gpurun_out/tune_53.jsonl; done; done
