cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "metrics or smoke or headline_size or fuzz" 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_48.txt
for b in 4 6; do ARA_METRICS_BLOCKS_PER_SM=$b timeout 300 python tools/time_metrics.py 2>&1 | tee -a gpurun_out/time_metrics_48.jsonl; done
