#!/usr/bin/env python3
"""Time the scan of small trial batches (the last partial round of a strong-scaling slice) under
tuning variants: which configuration finishes a few thousand 1000-event trials soonest on an
otherwise idle GPU?  (Tuning aid.)  Variants are KEY=VAL;KEY=VAL environment sets read at
ara_set_layers; ARA_LIB_VARIANT selects a tuning library.  Prints one JSON line per (n, variant)."""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="2000,5000,11336,20000,28416")
    ap.add_argument("--variants", default="base@")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch

    from paper_1308_2572_b200 import ara
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    spec = datagen.PRESETS["headline"].replace(n_trials=max(int(x) for x in args.n.split(",")))
    ds = datagen.generate(spec)
    d_off_all = torch.from_numpy(ds.trial_offsets.view(np.int64)).to(dev).view(torch.uint64)
    d_ids = torch.from_numpy(ds.events.view(np.int32)).to(dev).view(torch.uint32)
    ref = {}
    for v in args.variants.split(","):
        name, envs = v.split("@", 1)
        for kv in envs.split(";"):
            if kv:
                k, val = kv.split("=", 1)
                os.environ[k] = val
        ctx = ara.Context(0, stream)
        ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses,
                          ds.fin)
        ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
        for n in (int(x) for x in args.n.split(",")):
            ylt = torch.empty((1, n), dtype=torch.float64, device=dev)
            off = d_off_all[:n + 1]
            for _ in range(3):
                ctx.ara_run(off, d_ids, ylt)
            ctx.ara_synchronize()
            ts = []
            for _ in range(args.reps):
                a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.ara_run(off, d_ids, ylt)
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            out = ylt.cpu().numpy()
            same = bool(np.array_equal(out, ref.setdefault(n, out)))
            print(json.dumps({"variant": name, "lib": os.environ.get("ARA_LIB_VARIANT", ""),
                              "n": n, "ms": float(np.median(ts)),
                              "kernel": ctx.ara_get_info().last_kernel.decode(),
                              "same_as_first": same}), flush=True)
        ctx.close()
        for kv in envs.split(";"):
            if kv:
                os.environ.pop(kv.split("=", 1)[0], None)


if __name__ == "__main__":
    main()
