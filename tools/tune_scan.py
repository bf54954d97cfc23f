#!/usr/bin/env python3
"""Time scan-kernel variants on one workload in one process (tuning aid, not a bench line).

Variants are selected through the library's tuning environment variables (read at
ara_set_layers): ARA_SCAN_GROUP (lanes per trial for 16-column rows) and ARA_SCAN_MINB
(__launch_bounds__ min blocks).  Every variant's YLT must equal the first variant's bit for bit.
Prints one JSON line per variant.
"""
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
    ap.add_argument("--config", default="headline")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--variants", default="2:0,4:0,1:0",
                    help="comma list of G:MINB[:MAPMODE], or name@KEY=VAL;KEY=VAL (env only)")
    ap.add_argument("--flags", type=int, default=0, help="ara_run flags (4 = ARA_RUN_BALANCE)")
    ap.add_argument("--sched", default="", help="ARA_SCAN_SCHED: static | dynamic")
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--env", action="append", default=[], help="KEY=VALUE set before the runs")
    args = ap.parse_args()
    import torch

    from paper_1308_2572_b200 import ara
    for kv in args.env:
        k, v = kv.split("=", 1)
        os.environ[k] = v
    spec = datagen.PRESETS[args.config]
    ds = datagen.generate(spec)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    d_off = torch.from_numpy(ds.trial_offsets.view(np.int64)).to(dev).view(torch.uint64)
    d_ids = torch.from_numpy(ds.events.view(np.int32)).to(dev).view(torch.uint32)
    E = spec.elts_per_layer
    n, n_ev = ds.n_trials, int(ds.trial_offsets[-1])
    L = ds.n_layers
    bytes_alg = n_ev * (4 + args.precision // 8 * E * L) + 8 * n * L + 8 * (n + 1)
    ref = None
    for v in args.variants.split(","):
        if "@" in v:  # name@KEY=VAL;KEY=VAL: tuning environment only
            for kv in v.split("@", 1)[1].split(";"):
                if kv:
                    k, val = kv.split("=", 1)
                    os.environ[k] = val
        else:
            g, mb, *mm = v.split(":")  # G:MINB[:ARA_MAP_MODE]
            os.environ["ARA_SCAN_GROUP"] = g
            os.environ["ARA_SCAN_MINB"] = mb
            if mm:
                os.environ["ARA_MAP_MODE"] = mm[0]
        os.environ["ARA_SCAN_SCHED"] = args.sched
        ctx = ara.Context(0, stream)
        ctx.ara_set_precision(args.precision)
        ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses,
                          ds.fin)
        ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
        ylt = torch.empty((ds.n_layers, n), dtype=torch.float64, device=dev)
        for _ in range(3):
            ctx.ara_run(d_off, d_ids, ylt, flags=args.flags)
        ctx.ara_synchronize()
        ts = []
        for _ in range(args.reps):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.ara_run(d_off, d_ids, ylt, flags=args.flags)
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ctx.ara_synchronize()
        out = ylt.cpu().numpy()
        same = True if ref is None else bool(np.array_equal(out, ref))
        ref = out if ref is None else ref
        ms = float(np.median(ts))
        import hashlib
        print(json.dumps({"variant": v, "lib": os.environ.get("ARA_LIB_VARIANT", ""),
                          "ylt_sha1": hashlib.sha1(out.tobytes()).hexdigest()[:16],
                          "env": args.env, "sched": args.sched or f"flags={args.flags}",
                          "config": args.config, "ms_median": ms,
                          "ms_min": float(min(ts)), "GBps_alg": bytes_alg / ms / 1e6,
                          "trial_events_per_s": n_ev * ds.n_layers / ms * 1e3,
                          "same_as_first": same}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
