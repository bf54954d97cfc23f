cd $GRAFT_REPO_ROOT
timeout 600 python tools/sanitize_cases.py 2>&1 | tail -2 | tee gpurun_out/sanitize_plain_34.txt
timeout 1200 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_cases.py > gpurun_out/sanitizer_memcheck_34.txt 2>&1; tail -4 gpurun_out/sanitizer_memcheck_34.txt
timeout 1200 compute-sanitizer --tool racecheck python tools/sanitize_cases.py > gpurun_out/sanitizer_racecheck_34.txt 2>&1; tail -3 gpurun_out/sanitizer_racecheck_34.txt
timeout 1200 compute-sanitizer --tool initcheck python tools/sanitize_cases.py > gpurun_out/sanitizer_initcheck_34.txt 2>&1; tail -3 gpurun_out/sanitizer_initcheck_34.txt
timeout 900 python bench.py --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_34_portfolio.json 2>/dev/null
ARA_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config medium --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_34_n2_same_gpu.json 2> gpurun_out/bench_34_n2.err; tail -2 gpurun_out/bench_34_n2.err; cat gpurun_out/bench_34_n2_same_gpu.json | cut -c1-300
