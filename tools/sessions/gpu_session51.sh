cd $GRAFT_REPO_ROOT
for lib in pf0 "" pf12; do
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_51.jsonl
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 3 2>/dev/null | tee -a gpurun_out/tune_51.jsonl
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config sweep-ragged --variants 0:0:2 --reps 5 2>/dev/null | tee -a gpurun_out/tune_51.jsonl
done
