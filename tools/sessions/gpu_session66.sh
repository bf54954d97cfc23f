# Session 66: 8M-entry metrics at extreme probabilities.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "metrics_8m" -rs --durations=3 2>&1 | tail -25 | tee gpurun_out/pytest_66.txt
