#!/usr/bin/env python3
"""One-GPU emulation of the strong-scaling split of the headline workload (one fixed
1M x 1000 workload decomposed over 1/2/4/8 GPUs).

For R in 1, 2, 4, 8 this times, on this one GPU, exactly what rank 0 of an R-rank run computes per
step: the scan of its contiguous slice (n/R trials, dist.partition_trials) and PML/TVaR over the
whole gathered n-entry YLT (every rank computes the metrics after the all-gather); and bench.py's
default split, in which rank 0 alone computes the metrics and scans correspondingly fewer trials
(dist.partition_rank0_offload): the step is then the slower of rank 0 (its slice + the metrics)
and the other ranks (their slices).  The all-gather
itself cannot run on one GPU; it is reported from a bandwidth model (n*8 bytes over NVLink at the
B200_PROFILING.md peer figure of 770 GB/s per direction, i.e. an upper bound on its cost) and
kept separate.  Each slice's YLT is checked against the whole run's YLT (bit-identical).
Prints one JSON line per R.

    python tools/strong_emulation.py [--config headline] [--reps 10]
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
    args = ap.parse_args()
    import torch

    from paper_1308_2572_b200 import ara
    from paper_1308_2572_b200.dist import partition_rank0_offload, partition_trials
    spec = datagen.PRESETS[args.config]
    ds = datagen.generate(spec)
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)
    ctx = ara.Context(0, stream)
    ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses, ds.fin)
    ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
    n, L = ds.n_trials, ds.n_layers
    d_off_all = torch.from_numpy(ds.trial_offsets.view(np.int64)).to(dev).view(torch.uint64)
    d_ids = torch.from_numpy(ds.events.view(np.int32)).to(dev).view(torch.uint32)
    full = torch.empty((L, n), dtype=torch.float64, device=dev)
    for _ in range(3):
        ctx.ara_run(d_off_all, d_ids, full)
    ctx.ara_synchronize()
    p = [1 - 1 / rp for rp in (10, 25, 50, 100, 250, 500, 1000)]

    def time_slice(a, b, metrics):
        """Median scan time of trials [a, b) (and of the metrics over the n gathered entries);
        the slice's YLT must equal the whole run's."""
        off = d_off_all[a:b + 1]
        ev0 = int(ds.trial_offsets[a])
        ylt = torch.empty((L, b - a), dtype=torch.float64, device=dev)
        for _ in range(3):  # warm-up (length / hit verdicts settle)
            ctx.ara_run(off, d_ids[ev0:], ylt)
        ctx.ara_synchronize()
        scan, met = [], []
        for _ in range(args.reps):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream)
            ctx.ara_run(off, d_ids[ev0:], ylt)
            e[1].record(stream)
            if metrics:
                ctx.ara_metrics_rows(full, p)
            e[2].record(stream)
            e[2].synchronize()
            scan.append(e[0].elapsed_time(e[1]))
            met.append(e[1].elapsed_time(e[2]))
        ctx.ara_synchronize()
        return (float(np.median(scan)), float(np.median(met)) if metrics else 0.0,
                bool(torch.equal(ylt, full[:, a:b])))

    base = None
    for R in (1, 2, 4, 8):
        # every rank computes the metrics, trials split evenly (bench.py --no-offload)
        a, b = partition_trials(n, R)[0]
        sm, mm, same = time_slice(a, b, True)
        gather_ms = 0.0 if R == 1 else (R - 1) / R * n * 8 * L / 770e9 * 1e3
        step = sm + mm + gather_ms
        if base is None:
            base = step
        # bench.py default for R > 1: rank 0 alone computes the metrics and scans mu fewer
        # trials (mu = the metrics' cost in scanned trials, measured as bench.py does)
        mu = mm / (sm / (b - a)) if R > 1 else 0.0
        parts = partition_rank0_offload(n, R, mu)
        s0, m0, same0 = time_slice(parts[0][0], parts[0][1], True)
        s1, _, same1 = time_slice(parts[-1][0], parts[-1][1], False) if R > 1 else (s0, 0, True)
        step_off = max(s0 + m0, s1) + gather_ms
        ev = int(ds.trial_offsets[b] - ds.trial_offsets[a]) * L
        print(json.dumps({
            "R": R, "trials_per_gpu": b - a, "scan_ms": sm, "metrics_ms": mm,
            "allgather_model_ms": gather_ms, "step_ms": step,
            "trial_events_per_s_per_gpu": ev / (sm * 1e-3),
            "strong_efficiency_model": base / (R * step),
            "offload": {"mu_trials": mu, "trials_rank0": parts[0][1] - parts[0][0],
                        "trials_other": parts[-1][1] - parts[-1][0],
                        "rank0_scan_ms": s0, "rank0_metrics_ms": m0, "other_scan_ms": s1,
                        "step_ms": step_off, "strong_efficiency_model": base / (R * step_off)},
            "slice_bit_identical": same and same0 and same1,
            "kernel": ctx.ara_get_info().last_kernel.decode(), "config": args.config}),
            flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
