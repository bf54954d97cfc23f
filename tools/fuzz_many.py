#!/usr/bin/env python3
"""Run the GPU fuzz parity case (tests/test_parity_gpu.py::_fuzz_dataset) over many seeds:
full scan in map modes 0-2, hoisted scan, fp32 every third seed, portfolio kernels as the
portfolios allow -- every YLT bit-identical to the oracle.  Prints one summary JSON line.

    python tools/fuzz_many.py --seeds 300
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=300)
    ap.add_argument("--first", type=int, default=5000)
    args = ap.parse_args()
    import torch

    import oracle
    from paper_1308_2572_b200 import ara
    from tests import test_parity_gpu as T
    stream = torch.cuda.current_stream()
    runs, bad, kernels = 0, [], {}
    for seed in range(args.first, args.first + args.seeds):
        f32 = seed % 3 == 2
        ds = T._fuzz_dataset(seed, f32)
        os.environ["ARA_MAP_MODE"] = str(seed % 3)
        want = oracle.run_analysis(ds, n_threads=8, precision=32 if f32 else 64)
        ctx = ara.Context(0, stream)
        if f32:
            ctx.ara_set_precision(32)
        ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses,
                          ds.fin)
        ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
        info = ctx.ara_get_info()
        kernels[info.layer_kernel] = kernels.get(info.layer_kernel, 0) + 1
        flag_sets = [ara.ARA_RUN_SYNC, ara.ARA_RUN_SYNC]  # second run: stale-verdict choices
        if ds.n_layers <= 8:
            flag_sets.append(ara.ARA_RUN_SYNC | ara.ARA_RUN_HOIST)
        for fl in flag_sets:
            got = T.gpu_ylt(ds, stream, ctx=ctx, flags=fl)
            runs += 1
            same = (got == want) | (np.isnan(got) & np.isnan(want))
            if not same.all():
                bad.append({"seed": seed, "flags": fl, "n_bad": int((~same).sum())})
        ctx.close()
    print(json.dumps({"seeds": args.seeds, "runs": runs, "mismatches": bad,
                      "layer_kernels": kernels}), flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
