cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "bench_json or metrics" 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_47.txt
for b in 1 2 4; do ARA_METRICS_BLOCKS_PER_SM=$b timeout 300 python tools/time_metrics.py 2>&1 | tee -a gpurun_out/time_metrics_47.jsonl; done
timeout 600 ncu --set full --clock-control none -k regex:metrics_kernel -s 3 -c 1 -o gpurun_out/prof_metrics_47 python tools/time_metrics.py > /dev/null 2>&1
