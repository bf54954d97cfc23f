# Session 71: F4 outputs through the length-bucketed warp-batched kernels (BAL) instead of
# per-group tickets.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "f4 or stale or fuzz or extreme_length or dynamic_balance" 2>&1 | tail -3 | tee gpurun_out/pytest_71.txt
timeout 600 python tools/time_f4.py | tee gpurun_out/time_f4_71.json
ARA_SCAN_SCHED=dynamic timeout 600 python tools/time_f4.py | tee gpurun_out/time_f4_71_pergroup.json
