# Session 77: clock sampling with NVML (10 ms) in addition to nvidia-smi.
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_77.json 2> gpurun_out/bench_77.err; tail -3 gpurun_out/bench_77.err
timeout 900 python -m pytest tests/test_bench_contract.py -q 2>&1 | tail -2
