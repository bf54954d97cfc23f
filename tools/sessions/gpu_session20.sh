cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv | tee gpurun_out/smi_20.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_20.txt
timeout 600 python bench.py --steps 20 --warmup 3 --json-out gpurun_out/bench_20.json 2> gpurun_out/bench_20.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 3 -c 1 -o gpurun_out/prof_scan_20 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_20.log 2>&1
ncu -i gpurun_out/prof_scan_20.ncu-rep --page raw --csv > gpurun_out/prof_scan_20_raw.csv 2>&1
ls -la gpurun_out | tail -12
