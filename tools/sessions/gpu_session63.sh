# Session 63: the id load shares its scoreboard with the next chunk's first row gather (SASS
# control bits), so every chunk's first event waits for the id stream's latency.  Variants:
# ids L1-allocating (idl1), + L1 prefetch 4/8 chunks ahead (idpf4/idpf8), id load at the top
# of the chunk iteration (idearly), both (idearlyl1).
cd $GRAFT_REPO_ROOT
for cfg in headline sweep-ragged; do
  for lib in "" idl1 idpf4 idpf8 idearly idearlyl1; do
    ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config $cfg --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_63_ids.jsonl
  done
done
for lib in "" idl1 idpf4 idearlyl1; do
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2 --reps 10 --env ARA_MAP_MODE=1 2>/dev/null | tee -a gpurun_out/tune_63_ids.jsonl
done
for lib in "" idl1 idpf4; do
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config portfolio --variants 0:0:2 --reps 3 2>/dev/null | tee -a gpurun_out/tune_63_ids.jsonl
done
