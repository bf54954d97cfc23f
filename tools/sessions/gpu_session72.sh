# Session 72: after the F4 schedule change: full GPU suite, smoke, sanitizers (memcheck, racecheck).
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_72.txt
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_cases.py > gpurun_out/sanitizer_memcheck_72.txt 2>&1; tail -3 gpurun_out/sanitizer_memcheck_72.txt
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > gpurun_out/sanitizer_racecheck_72.txt 2>&1; tail -2 gpurun_out/sanitizer_racecheck_72.txt
