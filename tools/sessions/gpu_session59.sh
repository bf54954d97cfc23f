cd $GRAFT_REPO_ROOT
for lib in abl1 abl2 abl3 ""; do
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_59_ablation.jsonl
done
for lib in abl1 abl2 abl3 ""; do
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 3 --env ARA_PORTFOLIO=0 2>/dev/null | tee -a gpurun_out/tune_59_ablation.jsonl
done
