set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
nproc; lscpu | grep -E "Model name|^CPU\(s\)"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 | tee gpurun_out/pytest_gpu_1.txt
timeout 600 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_1.json 2> gpurun_out/bench_1.err
tail -5 gpurun_out/bench_1.err
ARA_SCAN_GROUP=2 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null > gpurun_out/bench_g2.json
ARA_SCAN_GROUP=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null > gpurun_out/bench_g1.json
cat gpurun_out/bench_g2.json gpurun_out/bench_g1.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_1.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_1 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_1.log 2>&1
tail -3 gpurun_out/ncu_1.log
