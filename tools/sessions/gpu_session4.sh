cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_4.txt
timeout 900 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_4.json 2> gpurun_out/bench_4.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_4.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:metrics_kernel -s 3 -c 1 -o gpurun_out/prof_metrics_4 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_4m.log 2>&1
tail -2 gpurun_out/ncu_4.log gpurun_out/ncu_4m.log
