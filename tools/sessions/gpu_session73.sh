# Session 73: F4 increments staged per 8-event chunk and stored as 64-byte segments.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_parity_gpu.py -x -q -k "f4 or stale or fuzz or extreme_length or dynamic_balance" 2>&1 | tail -3 | tee gpurun_out/pytest_73.txt
timeout 600 python tools/time_f4.py | tee gpurun_out/time_f4_73.json
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > gpurun_out/sanitizer_racecheck_73.txt 2>&1; tail -2 gpurun_out/sanitizer_racecheck_73.txt
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_cases.py > gpurun_out/sanitizer_memcheck_73.txt 2>&1; tail -2 gpurun_out/sanitizer_memcheck_73.txt
