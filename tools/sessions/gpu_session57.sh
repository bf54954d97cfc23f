cd $GRAFT_REPO_ROOT
for lib in "" hl1; do
ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2 --reps 10 --flags 8 2>/dev/null | tee -a gpurun_out/tune_57.jsonl
ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config sweep-h10 --variants 0:0:2 --reps 10 --flags 8 2>/dev/null | tee -a gpurun_out/tune_57.jsonl
done
