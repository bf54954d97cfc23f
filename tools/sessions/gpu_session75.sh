# Session 75: F4 increment kernel at 2 blocks/SM (no register cap, no spills) vs 3.
cd $GRAFT_REPO_ROOT
for lib in "" f4m2; do ARA_LIB_VARIANT=$lib timeout 600 python tools/time_f4.py | sed "s/^{/{\"lib\": \"$lib\", /" | tee -a gpurun_out/time_f4_75.jsonl; done
