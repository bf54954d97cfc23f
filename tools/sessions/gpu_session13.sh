cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_13.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke_13.txt
timeout 900 compute-sanitizer --tool memcheck --leak-check full python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_memcheck.txt 2>&1; tail -4 gpurun_out/sanitizer_memcheck.txt
timeout 900 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.txt 2>&1; tail -3 gpurun_out/sanitizer_racecheck.txt
timeout 900 compute-sanitizer --tool initcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_initcheck.txt 2>&1; tail -3 gpurun_out/sanitizer_initcheck.txt
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_13.json 2> gpurun_out/bench_13.err
ARA_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_13_n2.json 2> gpurun_out/bench_13_n2.err
timeout 600 python bench.py --config sweep-ragged --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_13_ragged.json 2>/dev/null
timeout 900 python bench.py --config portfolio --steps 5 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_13_portfolio.json 2>/dev/null
timeout 600 python bench.py --precision 32 --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_13_f32.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_13_ref.json 2> gpurun_out/bench_13_ref.err
ls -la gpurun_out | tail -20
