# Session 69: more resident warps for the map-mode 0/1 scan launches: 32/64-thread blocks with
# register caps (__maxnreg__) 136-152 instead of 128-thread blocks at 168 registers (12 warps/SM).
cd $GRAFT_REPO_ROOT
for lib in "" t64 t64n152 t64n144 t64n136 t32n152 t32n144 t32n136 t64b1; do
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config headline --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_69_occupancy.jsonl
done
for lib in "" t32n152 t32n144; do
  ARA_LIB_VARIANT=$lib timeout 300 python tools/tune_scan.py --config sweep-ragged --variants 0:0:2 --reps 10 2>/dev/null | tee -a gpurun_out/tune_69_occupancy.jsonl
done
