# Session 76: final round-1 check: build, smoke, full GPU suite, default bench line.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_76.txt
timeout 600 python bench.py > gpurun_out/bench_76.json 2> gpurun_out/bench_76.err; tail -c 300 gpurun_out/bench_76.json
