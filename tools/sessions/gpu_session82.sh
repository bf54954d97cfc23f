# Session 82: the multi-rank bench path (2 ranks sharing one GPU over gloo) on the final bench.py.
cd $GRAFT_REPO_ROOT
ARA_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config medium --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_2rank_82.json 2> gpurun_out/bench_2rank_82.err; echo rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_2rank_82.json')); print(d['n_gpus'], d['ms_per_step'], d['clocks']['samples'], d['e2e']['ms_per_step'], d['config']['parallelism'])"
ARA_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --impl reference --config medium --steps 1 --warmup 3 > gpurun_out/bench_2rank_ref_82.json 2>&1; echo rc=$?; tail -c 200 gpurun_out/bench_2rank_ref_82.json
