cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x --durations=12 2>&1 | tail -22 | tee gpurun_out/pytest_gpu_33.txt
timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2,0:0:1 --reps 5 2>/dev/null | tee gpurun_out/tune_33.jsonl
timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2,0:0:1 --reps 5 --env ARA_PORTFOLIO_SHFL=0 2>/dev/null | tee -a gpurun_out/tune_33.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:portfolio_kernel -s 1 -c 1 -o gpurun_out/prof_portfolio_33 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 1 > /dev/null 2>&1
ls gpurun_out | tail -5
