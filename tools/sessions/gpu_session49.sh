cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2 | tee gpurun_out/pytest_gpu_49.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | tee gpurun_out/smoke_49.txt
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_49.json 2> gpurun_out/bench_49.err | cut -c1-150
timeout 900 python bench.py --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_49_portfolio.json 2>/dev/null | cut -c1-150
timeout 600 python bench.py --config sweep-ragged --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --json-out gpurun_out/bench_49_ragged.json 2>/dev/null | cut -c1-150
timeout 600 python bench.py --precision 32 --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_49_f32.json 2>/dev/null | cut -c1-150
timeout 900 python bench.py --hoist --steps 20 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_49_hoist.json 2>/dev/null | cut -c1-150
timeout 900 python bench.py --hoist --config portfolio --steps 10 --warmup 3 --no-cpu-baseline --json-out gpurun_out/bench_49_hoist_portfolio.json 2>/dev/null | cut -c1-150
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_49_ref.json 2> gpurun_out/bench_49_ref.err
ARA_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config medium --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_49_n2_same_gpu.json 2> gpurun_out/bench_49_n2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_49.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_49_hoist.csv python bench.py --hoist --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_49 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out | grep _49
