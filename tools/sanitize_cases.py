#!/usr/bin/env python3
"""Small runs of every kernel path, for compute-sanitizer (memcheck / racecheck / initcheck):

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py

single layer (map modes 0-2), the pair scans of every row width (16-64 columns),
multi-layer per-layer rows, union rows with the shared F row and
with register shuffles, F4 outputs, fp32, host-buffer run, PML/TVaR, the hoisted scan, and the
runs that follow the previous run's length / hit-probe verdicts (identity order, mode-1 body).  Each YLT is checked against
the oracle (test infrastructure), so a run that passes under the sanitizer is also correct."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402


def main():
    import torch

    from paper_1308_2572_b200 import ara
    dev = torch.device("cuda:0")
    stream = torch.cuda.current_stream(dev)

    def run(ds, precision=64, env=(), outputs=False):
        for k, v in env:
            os.environ[k] = v
        ctx = ara.Context(0, stream)
        ctx.ara_set_precision(precision)
        ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses,
                          ds.fin)
        ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
        for k, _ in env:
            del os.environ[k]
        off = torch.from_numpy(ds.trial_offsets.view(np.int64)).to(dev).view(torch.uint64)
        ev = torch.from_numpy(ds.events.view(np.int32)).to(dev).view(torch.uint32)
        L, n = ds.n_layers, ds.n_trials
        ylt = torch.empty((L, n), dtype=torch.float64, device=dev)
        if outputs:
            mo = torch.empty((L, n), dtype=torch.float64, device=dev)
            inc = torch.empty((L, int(ds.trial_offsets[-1])), dtype=torch.float64, device=dev)
            ctx.ara_run_outputs(off, ev, ylt, d_max_occ=mo, d_event_inc=inc, flags=ara.ARA_RUN_SYNC)
        else:
            # three runs: the later ones use the previous runs' length / hit verdicts (identity
            # order, mode-1 body), then the hoisted scan
            for fl in (ara.ARA_RUN_SYNC | ara.ARA_RUN_VALIDATE, ara.ARA_RUN_SYNC):
                ctx.ara_run(off, ev, ylt, flags=fl)
            got = ylt.cpu().numpy()
            if L <= 8:
                ctx.ara_run(off, ev, ylt, flags=ara.ARA_RUN_SYNC | ara.ARA_RUN_HOIST)
                assert np.array_equal(ylt.cpu().numpy(), got), "hoisted YLT differs"
        got = ylt.cpu().numpy()
        info = ctx.ara_get_info()
        pml, tvar = ctx.ara_metrics(ylt[0], [0.9, 0.99])
        h = np.empty((L, n))
        ctx.ara_run_host(ds.trial_offsets, ds.events, h)
        ctx.close()
        want = oracle.run_analysis(ds, n_threads=8, precision=precision)
        assert np.array_equal(got, want) and np.array_equal(h, want), "YLT mismatch"
        opml, _ = oracle.metrics(want[0], [0.9, 0.99])
        assert np.array_equal(pml, opml)
        return info

    tiny = datagen.PRESETS["tiny"].replace(n_trials=300, k_min=0, k_max=40)
    run(datagen.generate(tiny.replace(k_min=24, k_max=24)))  # equal lengths: identity order
    run(datagen.generate(datagen.PRESETS["tiny"].replace(n_trials=200, k_min=16, k_max=16,
                                                         hit=1.0)))  # all present: mode-1 body
    for mode in ("0", "1", "2"):
        run(datagen.generate(tiny), env=[("ARA_MAP_MODE", mode)])
    run(datagen.generate(tiny), outputs=True)
    run(datagen.generate(tiny), precision=32)
    # pair scans of every row width (W = 16 / 24 / 32 / 48 / 64: 2-4 lanes, interleaved rows),
    # plain and with F4 outputs, ragged lengths
    for e in (16, 20, 32, 40, 64):
        wide = tiny.replace(n_elts=e, elts_per_layer=e, k_min=0, k_max=30, seed=11 + e)
        run(datagen.generate(wide))
        run(datagen.generate(wide), outputs=True)
    pf = datagen.PRESETS["portfolio"].replace(n_trials=200, k_min=0, k_max=60,
                                              catalogue_size=100_000, pool_size=2000,
                                              records_per_elt=1000)
    assert run(datagen.generate(pf)).layer_kernel == 3
    assert run(datagen.generate(pf), env=[("ARA_PORTFOLIO_SHFL", "2")]).layer_kernel == 2
    assert run(datagen.generate(pf), env=[("ARA_PORTFOLIO_SHFL", "0")]).layer_kernel == 1
    assert run(datagen.generate(pf), env=[("ARA_PORTFOLIO", "0")]).layer_kernel == 0
    run(datagen.generate(pf), outputs=True)
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
