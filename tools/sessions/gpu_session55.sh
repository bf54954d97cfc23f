cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "sharded or metrics or c_example" 2>&1 | tail -3
for m in gather sharded; do
ARA_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config medium --steps 5 --warmup 3 --no-cpu-baseline --metrics $m > gpurun_out/bench_55_n2_$m.json 2> gpurun_out/bench_55_n2_$m.err; tail -1 gpurun_out/bench_55_n2_$m.err | cut -c1-200
python3 -c "import json; d=json.load(open('gpurun_out/bench_55_n2_$m.json')); print('$m', d['ms_per_step'], d['pml'], d['tvar'])"
done
