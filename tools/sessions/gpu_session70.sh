# Session 70: round-end check on the final code: build, smoke, full GPU suite, default bench.
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_70.txt 2>&1; echo "smoke rc=$?" | tee -a gpurun_out/smoke_70.txt
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_70.txt
timeout 600 python bench.py > gpurun_out/bench_70.json 2> gpurun_out/bench_70.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_70.json 2>&1
