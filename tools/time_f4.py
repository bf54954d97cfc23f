#!/usr/bin/env python3
"""Time ara_run_outputs (F4: per-trial max occurrence loss, per-event incremental losses) at the
headline size against plain ara_run (results are checked equal; timing aid)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402


def main():
    import torch

    from paper_1308_2572_b200 import ara
    spec = datagen.PRESETS["headline"]
    ds = datagen.generate(spec)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    off = torch.from_numpy(ds.trial_offsets.view(np.int64)).to(dev).view(torch.uint64)
    ids = torch.from_numpy(ds.events.view(np.int32)).to(dev).view(torch.uint32)
    n, n_ev = ds.n_trials, int(ds.trial_offsets[-1])
    ctx = ara.Context(0, stream)
    ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses, ds.fin)
    ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
    ylt = torch.empty((1, n), dtype=torch.float64, device=dev)
    ylt2 = torch.empty((1, n), dtype=torch.float64, device=dev)
    mo = torch.empty((1, n), dtype=torch.float64, device=dev)
    inc = torch.empty((1, n_ev), dtype=torch.float64, device=dev)

    def t(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    out = {"run_ms": t(lambda: ctx.ara_run(off, ids, ylt)),
           "outputs_max_occ_ms": t(lambda: ctx.ara_run_outputs(off, ids, ylt2, mo)),
           "outputs_max_occ_inc_ms": t(lambda: ctx.ara_run_outputs(off, ids, ylt2, mo, inc))}
    out["ylt_equal"] = bool(torch.equal(ylt, ylt2))
    out["inc_bytes"] = n_ev * 8
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
