cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_60.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py 2> gpurun_out/bench_60.err | tee gpurun_out/bench_60.json | cut -c1-200
timeout 900 python bench.py --impl reference 2>/dev/null | cut -c1-200
