#!/usr/bin/env python3
"""Calibrate the layer-term multipliers of datagen.PRESETS (run once; results pasted there).

Calls only datagen (inputs) and oracle/ (the CPU oracle).  For a preset and seed it
  1. runs every pool event as a one-event trial with identity layer terms, so the oracle's
     YLT entry is that event's combined loss lo(e) (Alg. 1 lines 4-13);
  2. sets OccR = q50(lo), OccL = q95(lo) - q50(lo)  (~50% of pool occurrences below the
     occurrence retention, ~5% at the occurrence limit);
  3. with those occurrence terms and AggR = 0, AggL = +inf runs the first 1,000 trials, so
     the YLT entry is the trial's occurrence-capped sum S, and sets AggR = q30(S),
     AggL = q_top(S) - q30(S)  (~30% of trials pay 0; top = 0.9995 by default, so ~0.05% pay
     the aggregate limit and PML/TVaR at the return periods 10-1000 years, p = 0.9-0.999, fall
     below the cap -- with top = 0.9 every one of them equalled AggL);
  4. prints the multipliers relative to the generator's scale M (and k_mean * M).
"""
import argparse
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import oracle  # noqa: E402


def q(v, p):
    s = np.sort(v)
    return float(s[min(max(int(math.ceil(p * len(s))) - 1, 0), len(s) - 1)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("preset", nargs="+")
    ap.add_argument("--trials", type=int, default=100_000)
    ap.add_argument("--top", type=float, default=0.9995)
    args = ap.parse_args()
    for name in args.preset:
        spec = datagen.PRESETS[name].replace(n_layers=1, occ_ret_m=1.0, occ_lim_m=1.0,
                                             agg_ret_m=1.0, agg_lim_m=1.0)
        ds = datagen.generate(spec, with_yet=False)
        M = ds.layer_terms[0, 0]
        k_mean = 0.5 * (spec.k_min + spec.k_max)
        # 1. lo(e) for every pool event
        ds.trial_offsets = np.arange(spec.pool_size + 1, dtype=np.uint64)
        ds.events = ds.pool.copy()
        ds.layer_terms = np.array([[0.0, math.inf, 0.0, math.inf]])
        lo = oracle.run_analysis(ds, n_threads=os.cpu_count())[0]
        occ_r, occ_l = q(lo, 0.5), q(lo, 0.95) - q(lo, 0.5)
        # 3. S over the first trials
        off, ev = datagen.generate_yet(spec, ds.pool, 0, min(args.trials, spec.n_trials))
        ds.trial_offsets, ds.events = off, ev
        ds.layer_terms = np.array([[occ_r, occ_l, 0.0, math.inf]])
        S = oracle.run_analysis(ds, n_threads=os.cpu_count())[0]
        agg_r, agg_l = q(S, 0.3), q(S, args.top) - q(S, 0.3)
        print(f"{name}: occ_ret_m={occ_r / M:.4f}, occ_lim_m={occ_l / M:.4f}, "
              f"agg_ret_m={agg_r / (k_mean * M):.4f}, agg_lim_m={agg_l / (k_mean * M):.4f}")


if __name__ == "__main__":
    main()
