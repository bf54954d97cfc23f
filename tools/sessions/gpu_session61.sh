cd $GRAFT_REPO_ROOT
timeout 1500 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_cases.py > gpurun_out/sanitizer_memcheck_61.txt 2>&1; tail -3 gpurun_out/sanitizer_memcheck_61.txt
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > gpurun_out/sanitizer_racecheck_61.txt 2>&1; tail -2 gpurun_out/sanitizer_racecheck_61.txt
timeout 1500 compute-sanitizer --tool initcheck python tools/sanitize_cases.py > gpurun_out/sanitizer_initcheck_61.txt 2>&1; tail -2 gpurun_out/sanitizer_initcheck_61.txt
timeout 1500 compute-sanitizer --tool synccheck python tools/sanitize_cases.py > gpurun_out/sanitizer_synccheck_61.txt 2>&1; tail -2 gpurun_out/sanitizer_synccheck_61.txt
