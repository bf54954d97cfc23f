# Session 65: extreme trial-length skew parity test.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "extreme_length_skew or catalogue_at_max" -rs --durations=5 2>&1 | tail -15 | tee gpurun_out/pytest_65.txt
