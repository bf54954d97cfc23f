cd $GRAFT_REPO_ROOT
./tools/microbench_rowpattern 262144 1000 | tee gpurun_out/microbench_rowpattern_27.jsonl
for m in 1 2; do
timeout 300 python tools/tune_scan.py --config headline --variants 0:0:$m,4:0:$m,4:4:$m --reps 5 --env ARA_SCAN_DEPTH=4 2>&1
timeout 300 python tools/tune_scan.py --config headline --variants 4:0:$m --reps 5 --env ARA_SCAN_DEPTH=8 2>&1
done | tee gpurun_out/tune_27.jsonl
