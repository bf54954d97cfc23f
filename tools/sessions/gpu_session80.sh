# Session 80: bench flag combinations after the e2e / clock edits.
cd $GRAFT_REPO_ROOT
for a in "--config portfolio --steps 5" "--hoist --steps 5" "--precision 32 --steps 5" "--config sweep-ragged --steps 5 --no-e2e" "--config medium --steps 5 --scaling strong"; do
  timeout 600 python bench.py $a --warmup 3 --no-cpu-baseline > gpurun_out/b80.json 2> gpurun_out/b80.err
  echo "$a rc=$? $(python -c "import json; d=json.load(open('gpurun_out/b80.json')); print(round(d['ms_per_step'],2), d['clocks']['samples'], (d.get('e2e') or {}).get('ms_per_step'))" 2>&1 | tail -1)"
done | tee gpurun_out/bench_flags_80.txt
