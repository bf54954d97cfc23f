#!/usr/bin/env python3
"""Time ara_metrics (A9, PML/TVaR at the 7 return periods) on YLT rows of 1M-8M entries shaped
like the headline's (30% zeros, a concentrated positive bulk), for the multi-GPU weak-scaling
note in DESIGN.md (every rank computes the metrics of the gathered N x 1M-entry YLT)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1308_2572_b200 import ara
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    ctx = ara.Context(0, stream)
    P = [1 - 1 / rp for rp in (10, 25, 50, 100, 250, 500, 1000)]
    rng = np.random.default_rng(1)
    for n in (1_000_000, 2_000_000, 4_000_000, 8_000_000):
        v = rng.normal(1.0e6, 4.0e5, n).clip(0, 3.3e6)
        v[rng.random(n) < 0.3] = 0.0
        d = torch.from_numpy(v).to(dev)
        for _ in range(3):
            ctx.ara_metrics(d, P)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(20):
            ctx.ara_metrics(d, P)
        b.record(stream)
        torch.cuda.synchronize()
        print(json.dumps({"n": n, "ms_per_call": a.elapsed_time(b) / 20,
                          "blocks_per_sm": os.environ.get("ARA_METRICS_BLOCKS_PER_SM", "4")}),
              flush=True)
        # the sharded select on one rank (the reduction is a no-op): its local cost per call
        import time as _t
        for _ in range(2):
            ctx.ara_metrics_sharded(d, n, P, lambda t: None)
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        for _ in range(10):
            ctx.ara_metrics_sharded(d, n, P, lambda t: None)
        torch.cuda.synchronize()
        print(json.dumps({"n": n, "sharded_ms_per_call_1rank": (_t.perf_counter() - t0) * 100}),
              flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
