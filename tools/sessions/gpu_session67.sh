# Session 67: e2e with every host buffer pinned and one pass over the host offsets.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py > gpurun_out/bench_67.json 2> gpurun_out/bench_67.err
tail -c 600 gpurun_out/bench_67.json
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "run_host" 2>&1 | tail -2
