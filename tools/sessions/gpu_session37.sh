cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_37.txt
for lib in "" pfadd; do ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_37.jsonl; done
bash tools/sweep.sh gpurun_out/sweep_37.jsonl
wc -l gpurun_out/sweep_37.jsonl
