# Bench line of every sweep configuration; SWEEP_HOIST=1 adds the hoisted scan.
cd $GRAFT_REPO_ROOT
out=${1:-gpurun_out/sweep.jsonl}
for c in sweep-e4 sweep-e8 sweep-e16 sweep-e20 sweep-e24 sweep-e32 sweep-e48 sweep-e64 sweep-k500 sweep-k2000 sweep-ragged sweep-h10 sweep-n8m sweep-bigstore; do
  for h in "" ${SWEEP_HOIST:+--hoist}; do
    timeout 900 python bench.py --config $c $h --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 >> $out
  done
done
