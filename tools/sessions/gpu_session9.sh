cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_9.txt
for cfg in headline sweep-ragged; do timeout 300 python tools/tune_scan.py --config $cfg --variants 0:0 --reps 5; done | tee gpurun_out/tune_9.jsonl
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_ragged python tools/tune_scan.py --config sweep-ragged --variants 0:0 --reps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_head9 python tools/tune_scan.py --config headline --variants 0:0 --reps 1 > /dev/null 2>&1
ls gpurun_out/
