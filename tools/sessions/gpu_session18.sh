cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "multilayer or widths or leading or balance" 2>&1 | tail -2
for pf in 1 0; do timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0 --reps 5 --env ARA_PORTFOLIO=$pf; done | tee gpurun_out/tune_18.jsonl
