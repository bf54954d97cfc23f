# Session 79: F4 outputs at every row width, both schedules.
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -k "f4_outputs_widths" 2>&1 | tail -4 | tee gpurun_out/pytest_79.txt
