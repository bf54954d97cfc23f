"""The seeded generator (datagen/): determinism, substreams, shapes and ranges."""
import numpy as np

import datagen


def test_determinism_and_slices():
    spec = datagen.PRESETS["tiny"].replace(n_trials=500, k_min=3, k_max=17)
    a = datagen.generate(spec)
    b = datagen.generate(spec)
    for f in ("pool", "rec_event_ids", "rec_losses", "fin", "layer_terms", "trial_offsets",
              "events"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    # a slice generated alone equals the same slice of the full YET (per-trial substreams)
    off, ev = datagen.generate_yet(spec, a.pool, 123, 77, n_threads=3)
    base = int(a.trial_offsets[123])
    assert np.array_equal(off + base, a.trial_offsets[123:201])
    assert np.array_equal(ev, a.events[base:int(a.trial_offsets[200])])
    c = datagen.generate(spec.replace(seed=spec.seed + 1))
    assert not np.array_equal(a.events, c.events)


def test_shapes_and_ranges():
    spec = datagen.PRESETS["medium"].replace(n_trials=200)
    ds = datagen.generate(spec)
    assert ds.pool.shape == (spec.pool_size,) and len(set(ds.pool.tolist())) == spec.pool_size
    assert ds.pool.min() >= 1 and ds.pool.max() <= spec.catalogue_size
    R = spec.records_per_elt
    for j in range(spec.n_elts):
        ids = ds.rec_event_ids[j * R:(j + 1) * R]
        assert len(set(ids.tolist())) == R  # unique per ELT
        assert np.isin(ids, ds.pool).all()
    assert (ds.rec_losses >= spec.loss_min).all() and (ds.rec_losses <= spec.loss_max).all()
    assert (ds.fin[:, 0] > 0).all() and (ds.fin[:, 1] >= 0).all() and (ds.fin[:, 2] >= 0).all()
    assert np.isinf(ds.fin[0::2, 2]).all()
    assert (ds.layer_terms >= 0).all()
    assert ds.events.shape[0] == spec.n_trials * spec.k_min
    assert np.isin(ds.events, ds.pool).all()  # hit = 1
    assert np.array_equal(ds.trial_offsets, np.arange(201, dtype=np.uint64) * 1000)


def test_hit_fraction_and_multilayer():
    spec = datagen.PRESETS["tiny"].replace(n_trials=5000)
    ds = datagen.generate(spec)
    frac = np.isin(ds.events, ds.pool).mean()
    # misses can also land on pool ids: P = h + (1-h) F/C
    assert abs(frac - (0.5 + 0.5 * 200 / 1000)) < 0.02
    p = datagen.PRESETS["portfolio"].replace(n_trials=10)
    dp = datagen.generate(p)
    assert dp.n_layers == 8 and dp.elt_index.shape[0] == 128
    counts = np.bincount(dp.elt_index, minlength=64)
    assert (counts == 2).all()  # each ELT shared by 2 layers
    assert len({tuple(r) for r in dp.layer_terms.tolist()}) == 8
