# Session 81: default bench line + GPU bench contract test on the final bench.py.
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/bench_81.json 2> gpurun_out/bench_81.err; python -c "import json; d=json.load(open('gpurun_out/bench_81.json')); print(d['ms_per_step'], d['clocks'], d['e2e']['ms_per_step'])"
timeout 900 python -m pytest tests/test_bench_contract.py -q 2>&1 | tail -1
