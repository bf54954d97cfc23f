# Session 64: the maximum-id catalogue test (map sizes 2^31 and 2^32 - 1 entries).
cd $GRAFT_REPO_ROOT
free -g | tee gpurun_out/free_64.txt
nvidia-smi --query-gpu=memory.total,memory.used --format=csv | tee -a gpurun_out/free_64.txt
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "catalogue_at_max_ids" -rs --durations=5 2>&1 | tail -15 | tee gpurun_out/pytest_64.txt
