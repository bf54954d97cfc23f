# Session 68: PCIe ceiling for the e2e line.
cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_h2d.py | tee gpurun_out/time_h2d.jsonl
