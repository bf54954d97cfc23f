cd $GRAFT_REPO_ROOT
timeout 600 python tools/sanitize_cases.py 2>&1 | tail -2 | tee gpurun_out/sanitize_plain_54.txt
timeout 1500 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_cases.py > gpurun_out/sanitizer_memcheck_54.txt 2>&1; tail -4 gpurun_out/sanitizer_memcheck_54.txt
timeout 1500 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > gpurun_out/sanitizer_racecheck_54.txt 2>&1; tail -3 gpurun_out/sanitizer_racecheck_54.txt
timeout 1500 compute-sanitizer --tool initcheck python tools/sanitize_cases.py > gpurun_out/sanitizer_initcheck_54.txt 2>&1; tail -3 gpurun_out/sanitizer_initcheck_54.txt
timeout 1500 compute-sanitizer --tool synccheck python tools/sanitize_cases.py > gpurun_out/sanitizer_synccheck_54.txt 2>&1; tail -3 gpurun_out/sanitizer_synccheck_54.txt
