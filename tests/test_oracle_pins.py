"""Pins of the CPU oracle (oracle/) to things other than itself.

Each test checks the oracle against what the paper, SPEC's hand-derived examples or plain
mathematics fix: worked examples (tests/golden/spec_examples.json), the excess-of-loss interval
characterisation evaluated in exact rationals (tests/_util.py), closed forms, textbook special
cases, invariants, monotonicity, homogeneity, brute force on tiny inputs.  The mistakes these
catch: a dropped term (identity / brute force), a wrong sign or index (interval erosion, SPEC
examples), a transposed operand (min/max order, retention vs limit), the in-place reading of
lines 19/25 (counterexample), FMA contraction (separate-rounding test), thread partition
dependence (determinism).
"""
import itertools
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import datagen
import oracle
from tests._util import (INF, elt_dicts, golden_value, make_dataset, seg, trial_events,
                         trial_exact, trial_S_exact, xl)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# --------------------------------------------------------------------------- golden examples
@pytest.mark.parametrize("case", GOLD["financial_terms"], ids=lambda c: c["cite"][:12])
def test_spec_financial_terms(case):
    args = [golden_value(a) for a in case["args"]]
    assert oracle.apply_financial_terms(*args) == case["expected"], case["cite"]


@pytest.mark.parametrize("case", GOLD["occurrence_terms"], ids=lambda c: c["cite"][:12])
def test_spec_occurrence_terms(case):
    args = [golden_value(a) for a in case["args"]]
    assert oracle.apply_occurrence_terms(*args) == case["expected"], case["cite"]


@pytest.mark.parametrize("case", GOLD["aggregate_terms"], ids=lambda c: c["cite"][:12])
def test_spec_aggregate_terms(case):
    inc = oracle.apply_aggregate_terms(case["lo"], golden_value(case["agg_retention"]),
                                       golden_value(case["agg_limit"]))
    assert inc.tolist() == case["expected"], case["cite"]


def test_spec_run_analysis():
    g = GOLD["run_analysis"]
    ds = make_dataset(g["catalogue_size"],
                      [{"records": e["records"], "fin": [golden_value(v) for v in e["fin"]]}
                       for e in g["elts"]],
                      [{"elts": L["elts"], "terms": L["terms"]} for L in g["layers"]],
                      g["trials"])
    assert oracle.run_analysis(ds).tolist() == g["expected_ylt"], g["cite"]


def test_simultaneous_not_in_place_reading():
    """Reading R5: the in-place ascending execution of lines 19/25 gives 190 > T_AggL."""
    g = GOLD["in_place_reading_counterexample"]
    lo = [float(v) for v in g["lo"]]
    R, L = g["agg_retention"], g["agg_limit"]
    # literal in-place, ascending (the forbidden reading), written out for contrast
    a = lo[:]
    for d in range(len(a)):
        a[d] = sum(a[: d + 1])
    a = [min(max(v - R, 0), L) for v in a]
    for d in range(len(a)):
        a[d] = a[d] - (a[d - 1] if d else 0)
    assert sum(a) == g["in_place_sum"] and sum(a) > L
    assert sum(oracle.apply_aggregate_terms(lo, R, L)) == g["simultaneous_sum"]


@pytest.mark.parametrize("case", GOLD["metrics"], ids=lambda c: c["cite"][:12])
def test_spec_metrics(case):
    v = np.arange(1, 101, dtype=np.float64)
    pml, tvar = oracle.metrics(v[::-1].copy(), [case["p"]])
    assert pml[0] == case["pml"] and tvar[0] == case["tvar"], case["cite"]


def test_paper_counts():
    """a DAT has one slot per catalogue event (15 x 2M = 30M slots for a
    15-ELT layer); length C+1 (slot 0 unused)."""
    dat = oracle.build_dat(2_000_000, [5, 1_999_999], [1.5, 2.5])
    assert dat.shape[0] == 2_000_001 and np.count_nonzero(dat) == 2
    assert 15 * (dat.shape[0] - 1) == GOLD["paper_counts"]["dat_slots_15_elts_2M_catalogue"]
    assert 1000 * 1_000_000 * 15 == GOLD["paper_counts"]["lookups_1M_trials_1000_events_15_elts"]


# --------------------------------------------------------------------------- elementary terms
def test_financial_terms_is_xl_layer_exhaustive():
    """F(x) = |[0, x*rate] cap [ret, ret+lim]| on a grid where fp64 is exact."""
    rates = [0.5, 1.0, 1.5, 2.0]
    for x in range(0, 41, 3):
        for rate in rates:
            for ret in [0, 1, 7, 20, 60]:
                for lim in [0, 1, 5, 30, INF]:
                    want = xl(Fraction(x) * Fraction(rate), Fraction(ret),
                              lim if lim == INF else Fraction(lim))
                    assert oracle.apply_financial_terms(x, rate, ret, lim) == want


def test_occurrence_terms_is_xl_layer_exhaustive():
    for lo in range(0, 61, 2):
        for r in [0, 1, 10, 33]:
            for L in [0, 4, 25, INF]:
                want = xl(Fraction(lo), Fraction(r), L if L == INF else Fraction(L))
                assert oracle.apply_occurrence_terms(lo, r, L) == want


def test_aggregate_terms_is_layer_erosion_random():
    """inc_d = |[S_{d-1}, S_d] cap [AggR, AggR+AggL]| exactly, on integer sequences."""
    rng = random.Random(7)
    for _ in range(500):
        k = rng.randint(0, 12)
        lo = [rng.choice([0, 0, rng.randint(0, 50)]) for _ in range(k)]
        R = rng.randint(0, 200)
        L = rng.choice([INF, rng.randint(0, 150)])
        inc = oracle.apply_aggregate_terms(lo, R, L)
        hi = INF if L == INF else R + L
        s = 0
        for d in range(k):
            assert inc[d] == seg(Fraction(s), Fraction(s + lo[d]), Fraction(R), hi)
            assert inc[d] >= 0
            s += lo[d]


# --------------------------------------------------------------------------- brute force
def _exhaustive_cases():
    rng = random.Random(1308)
    cat = 6
    for n_elts in (2, 3):
        elts = []
        for j in range(n_elts):
            members = rng.sample(range(1, cat + 1), rng.randint(2, cat))
            elts.append({e: rng.randint(1, 40) for e in members})
        fin = [(rng.choice([0.5, 1, 2]), rng.randint(0, 15), rng.choice([INF, rng.randint(0, 50)]))
               for _ in range(n_elts)]
        occ = (rng.randint(0, 20), rng.choice([INF, rng.randint(1, 60)]))
        agg = (rng.randint(0, 60), rng.choice([INF, rng.randint(1, 90)]))
        yield cat, elts, fin, occ, agg


@pytest.mark.parametrize("case_i", [0, 1])
def test_brute_force_every_trial_up_to_length_3(case_i):
    """Every trial of length 0..3 over a 6-event catalogue (repeats allowed) against the exact
    erosion formulation.  Integer/dyadic data: fp64 is exact, so equality is exact."""
    cat, elts, fin, occ, agg = list(_exhaustive_cases())[case_i]
    trials = [list(t) for k in range(4) for t in itertools.product(range(1, cat + 1), repeat=k)]
    ds = make_dataset(cat, [{"records": sorted(e.items()), "fin": f} for e, f in zip(elts, fin)],
                      [{"elts": list(range(len(elts))), "terms": (*occ, *agg)}], trials)
    ylt = oracle.run_analysis(ds)[0]
    for t, ev in enumerate(trials):
        assert ylt[t] == trial_exact(ev, elts, fin, occ, agg), (ev, ylt[t])


def test_brute_force_random_small_instances():
    """1,000 random instances, <= 5 events, <= 3 ELTs, catalogue <= 10."""
    rng = random.Random(2572)
    for _ in range(1000):
        cat = rng.randint(1, 10)
        n_elts = rng.randint(1, 3)
        elts = [{e: rng.randint(1, 30) for e in rng.sample(range(1, cat + 1), rng.randint(0, cat))}
                for _ in range(n_elts)]
        fin = [(rng.choice([0.25, 0.5, 1, 1.5, 2]), rng.randint(0, 10),
                rng.choice([INF, rng.randint(0, 40)])) for _ in range(n_elts)]
        occ = (rng.randint(0, 15), rng.choice([INF, rng.randint(0, 50)]))
        agg = (rng.randint(0, 50), rng.choice([INF, rng.randint(0, 80)]))
        ev = [rng.randint(1, cat) for _ in range(rng.randint(0, 5))]
        ds = make_dataset(cat, [{"records": sorted(e.items()), "fin": f}
                                for e, f in zip(elts, fin)],
                          [{"elts": list(range(n_elts)), "terms": (*occ, *agg)}], [ev])
        assert oracle.run_analysis(ds)[0, 0] == trial_exact(ev, elts, fin, occ, agg)


# --------------------------------------------------------------------------- closed forms
def test_closed_form_and_bounds_on_generated_data():
    """Telescoping: lr = min(max(S - AggR, 0), AggL) with S the exact
    occurrence-capped sum; fp64 error bounded by the rounding of S (absolute, since S - AggR
    may cancel: DESIGN.md tolerance derivation).  Bounds 0 <= lr <= AggL."""
    import datagen
    spec = datagen.PRESETS["tiny"].replace(n_trials=300, seed=42)
    ds = datagen.generate(spec)
    ylt = oracle.run_analysis(ds)[0]
    elts, fin = elt_dicts(ds, 0)
    occR, occL, aggR, aggL = ds.layer_terms[0]
    u = 2.0 ** -53
    for t in range(ds.n_trials):
        ev = trial_events(ds, t)
        S = trial_S_exact(ev, elts, fin, (occR, occL))
        exact = seg(Fraction(0), S, Fraction(aggR), Fraction(aggR) + Fraction(aggL))
        k, E = len(ev), len(elts)
        bound = 4 * (k + E + 2) * u * float(S + Fraction(aggR)) + 1e-300
        assert abs(ylt[t] - float(exact)) <= bound
        assert 0.0 <= ylt[t] <= aggL


def test_identity_terms_sum_raw_losses():
    """Identity terms (rate 1, retentions 0, limits absent): lr = sum of raw losses over the
    trial's events and the layer's ELTs (BASELINE.json north_star)."""
    rng = np.random.default_rng(3)
    cat = 50
    elts = [{int(e): int(rng.integers(1, 1000)) for e in rng.choice(np.arange(1, cat + 1), 30,
                                                                     replace=False)}
            for _ in range(4)]
    trials = [list(map(int, rng.integers(1, cat + 1, rng.integers(0, 40)))) for _ in range(50)]
    ds = make_dataset(cat, [{"records": sorted(e.items()), "fin": (1, 0, INF)} for e in elts],
                      [{"elts": [0, 1, 2, 3], "terms": (0, INF, 0, INF)}], trials)
    ylt = oracle.run_analysis(ds)[0]
    for t, ev in enumerate(trials):
        assert ylt[t] == sum(e.get(x, 0) for x in ev for e in elts)


def test_stop_loss_special_case():
    """One ELT, identity financial terms, OccR = 0, OccL = inf: the layer is an aggregate
    stop-loss, lr = min(max(sum x - AggR, 0), AggL)."""
    rng = np.random.default_rng(11)
    cat = 30
    elt = {int(e): int(rng.integers(1, 500)) for e in range(1, cat + 1)}
    trials = [list(map(int, rng.integers(1, cat + 1, rng.integers(0, 25)))) for _ in range(80)]
    for aggR, aggL in [(0, INF), (1000, 2000), (3000, 500), (10**6, 10)]:
        ds = make_dataset(cat, [{"records": sorted(elt.items()), "fin": (1, 0, INF)}],
                          [{"elts": [0], "terms": (0, INF, aggR, aggL)}], trials)
        ylt = oracle.run_analysis(ds)[0]
        for t, ev in enumerate(trials):
            tot = sum(elt[x] for x in ev)
            assert ylt[t] == min(max(tot - aggR, 0), aggL)


def test_per_occurrence_xl_special_case():
    """AggR = 0, AggL = inf: the layer is a per-occurrence XL, lr = sum_d min(max(x_d - OccR,
    0), OccL)."""
    rng = np.random.default_rng(12)
    cat = 30
    elt = {int(e): int(rng.integers(1, 500)) for e in range(1, cat + 1, 2)}
    trials = [list(map(int, rng.integers(1, cat + 1, rng.integers(0, 25)))) for _ in range(80)]
    ds = make_dataset(cat, [{"records": sorted(elt.items()), "fin": (1, 0, INF)}],
                      [{"elts": [0], "terms": (100, 250, 0, INF)}], trials)
    ylt = oracle.run_analysis(ds)[0]
    for t, ev in enumerate(trials):
        assert ylt[t] == sum(min(max(elt.get(x, 0) - 100, 0), 250) for x in ev)


# --------------------------------------------------------------------------- properties
def _small_int_dataset(seed, terms, fin_override=None):
    rng = random.Random(seed)
    cat = 20
    elts = [{e: rng.randint(1, 100) for e in rng.sample(range(1, cat + 1), 12)} for _ in range(3)]
    fin = fin_override or [(1, rng.randint(0, 20), rng.choice([INF, 60])) for _ in range(3)]
    trials = [[rng.randint(1, cat) for _ in range(rng.randint(0, 30))] for _ in range(40)]
    return make_dataset(cat, [{"records": sorted(e.items()), "fin": f} for e, f in zip(elts, fin)],
                        [{"elts": [0, 1, 2], "terms": terms}], trials)


def test_monotonicity():
    """lr non-increasing in OccR, AggR, retentions; non-decreasing in limits."""
    base = (10, 80, 200, 400)
    y0 = oracle.run_analysis(_small_int_dataset(5, base))[0]
    for i, sign in [(0, -1), (2, -1), (1, +1), (3, +1)]:
        for delta in (1, 7, 40):
            t = list(base); t[i] += delta
            y = oracle.run_analysis(_small_int_dataset(5, tuple(t)))[0]
            assert np.all(sign * (y - y0) >= 0), (i, delta)
    fin0 = [(1, 5, 60), (1, 0, INF), (1, 12, 60)]
    y0 = oracle.run_analysis(_small_int_dataset(5, base, fin0))[0]
    for bump in (1, 9):
        fin = [(1, 5 + bump, 60), (1, bump, INF), (1, 12 + bump, 60)]
        assert np.all(oracle.run_analysis(_small_int_dataset(5, base, fin))[0] <= y0)


def test_positive_homogeneity_bit_exact():
    """Scaling every loss and monetary term by 2^m scales lr by exactly 2^m;
    fails if any step contracts into an FMA or reorders a sum."""
    import datagen
    ds = datagen.generate(datagen.PRESETS["tiny"].replace(n_trials=200, seed=2572))
    y0 = oracle.run_analysis(ds)[0]
    for m in (-3, 5):
        c = 2.0 ** m
        ds2 = datagen.generate(datagen.PRESETS["tiny"].replace(n_trials=200, seed=2572))
        ds2.rec_losses = ds2.rec_losses * c
        ds2.fin = ds2.fin.copy(); ds2.fin[:, 1:] *= c
        ds2.layer_terms = ds2.layer_terms * c
        assert np.array_equal(oracle.run_analysis(ds2)[0], y0 * c)


def test_permutation_invariance_of_trial_total():
    """The trial total is invariant under reordering the trial's events (exact arithmetic);
    per-event increments are not.  fp64 within the rounding of S."""
    import datagen
    ds = datagen.generate(datagen.PRESETS["tiny"].replace(n_trials=200, seed=1308))
    y0 = oracle.run_analysis(ds)[0]
    rng = np.random.default_rng(0)
    ev = ds.events.copy()
    for t in range(ds.n_trials):
        a, b = int(ds.trial_offsets[t]), int(ds.trial_offsets[t + 1])
        ev[a:b] = rng.permutation(ev[a:b])
    y1 = oracle.run_analysis(ds, events=ev)[0]
    scale = ds.layer_terms[0, 2] + ds.layer_terms[0, 3]
    assert np.all(np.abs(y1 - y0) <= 64 * 2.0 ** -53 * scale)


def test_determinism_threads_and_selection():
    """bit-identical YLT for any worker count; a selection of trials equals the
    same columns of the full run (trials are independent)."""
    import datagen
    ds = datagen.generate(datagen.PRESETS["tiny"].replace(seed=42))
    y1 = oracle.run_analysis(ds, n_threads=1)
    for n in (2, 3, 8):
        assert np.array_equal(oracle.run_analysis(ds, n_threads=n), y1)
    sel = np.array([999, 0, 17, 17, 500], dtype=np.uint64)
    assert np.array_equal(oracle.run_analysis(ds, selection=sel), y1[:, sel.astype(np.int64)])


def test_absent_events_and_empty_trials():
    """Events absent from every ELT contribute 0; an empty trial
    gives 0."""
    ds = make_dataset(10, [{"records": [(1, 5.0)], "fin": (1, 0, INF)}],
                      [{"elts": [0], "terms": (0, INF, 0, INF)}], [[2, 3, 4], [], [1, 2, 1]])
    assert oracle.run_analysis(ds)[0].tolist() == [0.0, 0.0, 10.0]


def test_invalid_ids_rejected():
    """an id 0 or above the catalogue is a construction error."""
    with pytest.raises(ValueError):
        oracle.build_dat(10, [3, 11], [1.0, 1.0])
    with pytest.raises(ValueError):
        oracle.build_dat(10, [0], [1.0])
    ds = make_dataset(10, [{"records": [(1, 5.0)], "fin": (1, 0, INF)}],
                      [{"elts": [0], "terms": (0, INF, 0, INF)}], [[11]])
    with pytest.raises(ValueError):
        oracle.run_analysis(ds)


def test_dat_equals_compact_lookup():
    """direct-access lookup equals a compact (dict) lookup for every id."""
    rng = np.random.default_rng(5)
    for _ in range(100):
        C = int(rng.integers(1, 10_000))
        n = int(rng.integers(0, min(C, 500)))
        ids = rng.choice(np.arange(1, C + 1), n, replace=False).astype(np.uint32)
        ls = rng.uniform(0.5, 100.0, n)
        dat = oracle.build_dat(C, ids, ls)
        compact = dict(zip(ids.tolist(), ls.tolist()))
        assert dat.shape[0] == C + 1 and dat[0] == 0.0
        full = np.array([compact.get(e, 0.0) for e in range(1, C + 1)])
        assert np.array_equal(dat[1:], full)


# --------------------------------------------------------------------------- metrics
def test_metrics_against_numpy_and_brute_force():
    """Nearest-rank PML = numpy.quantile(method='inverted_cdf'); TVaR = mean of all v >= PML,
    brute force; TVaR >= PML; PML monotone in p."""
    rng = np.random.default_rng(9)
    ps = [0.5, 0.9, 0.96, 0.98, 0.99, 0.996, 0.998, 0.999]
    for _ in range(1000):
        n = int(rng.integers(1, 1000))
        v = np.round(rng.exponential(100.0, n)) * rng.choice([0, 1], n, p=[0.3, 0.7])
        pml, tvar = oracle.metrics(v, ps)
        for i, p in enumerate(ps):
            assert pml[i] == np.quantile(v, p, method="inverted_cdf")
            tail = v[v >= pml[i]]
            assert math.isclose(tvar[i], math.fsum(tail) / len(tail), rel_tol=1e-13)
            assert tvar[i] >= pml[i]
        assert np.all(np.diff(pml) >= 0)


def test_metrics_degenerate():
    pml, tvar = oracle.metrics(np.full(7, 3.5), [0.1, 0.99])
    assert pml.tolist() == [3.5, 3.5] and tvar.tolist() == [3.5, 3.5]
    pml, tvar = oracle.metrics(np.array([42.0]), [0.5])
    assert pml[0] == 42.0 and tvar[0] == 42.0
    with pytest.raises(ValueError):
        oracle.metrics(np.array([]), [0.5])
    for bad in (0.0, 1.0, -0.5, float("nan")):
        with pytest.raises(ValueError):
            oracle.metrics(np.array([1.0]), [bad])


def test_separate_rounding_no_fma():
    """Reading R7: x*rate and (.) - retention are each rounded to fp64 (no FMA).  CPython float
    arithmetic is IEEE 754 with separately rounded * and -, so it realises exactly that
    sequence; a contracted fma(x, rate, -ret) differs on a large share of random inputs."""
    rng = np.random.default_rng(77)
    x = rng.uniform(1e3, 1e8, 20000)
    rate = rng.uniform(0.8, 1.25, 20000)
    ret = x * rate * rng.uniform(0.0, 1.0, 20000)
    n_diff_from_exact = 0
    for xi, ri, ti in zip(x.tolist(), rate.tolist(), ret.tolist()):
        want = xi * ri - ti
        want = 0.0 if want < 0 else want
        got = oracle.apply_financial_terms(xi, ri, ti, math.inf)
        assert got == want
        n_diff_from_exact += float(Fraction(xi) * Fraction(ri) - Fraction(ti)) != got
    assert n_diff_from_exact > 1000  # the test data does exercise the double rounding


# --------------------------------------------------------------------------- F4 outputs
def test_event_increments_and_max_occurrence_brute_force():
    """F4 outputs, exactly on integer/dyadic data: the per-event increments of lines 24-26 are
    the erosion |[S_{d-1}, S_d] cap [AggR, AggR+AggL]| of each occurrence, they sum to lr
    (line 28), and max_occ is the largest occurrence loss xl(lo_d; OccR, OccL) of the trial
    (0 for an empty trial) -- the quantity whose distribution is the OEP curve."""
    cat, elts, fin, occ, agg = list(_exhaustive_cases())[1]
    trials = [list(t) for k in range(4) for t in itertools.product(range(1, cat + 1), repeat=k)]
    ds = make_dataset(cat, [{"records": sorted(e.items()), "fin": f} for e, f in zip(elts, fin)],
                      [{"elts": list(range(len(elts))), "terms": (*occ, *agg)}], trials)
    ylt, mo, inc = oracle.run_analysis(ds, outputs=True)
    agg_hi = INF if agg[1] == INF else Fraction(agg[0]) + Fraction(agg[1])
    for t, ev in enumerate(trials):
        pos = int(ds.trial_offsets[t])
        s_prev, best = Fraction(0), Fraction(0)
        for d, e in enumerate(ev):
            lo = sum((xl(Fraction(elts[j].get(e, 0)) * Fraction(fin[j][0]), Fraction(fin[j][1]),
                         fin[j][2] if fin[j][2] == INF else Fraction(fin[j][2]))
                      for j in range(len(elts))), Fraction(0))
            oc = xl(lo, Fraction(occ[0]), occ[1] if occ[1] == INF else Fraction(occ[1]))
            assert inc[0, pos + d] == seg(s_prev, s_prev + oc, Fraction(agg[0]), agg_hi)
            s_prev += oc
            best = max(best, oc)
        assert mo[0, t] == best
        assert ylt[0, t] == math.fsum(inc[0, pos:pos + len(ev)])
    # selection keeps event positions of the whole YET
    sel = np.array([5, 2], np.uint64)
    y2, m2, i2 = oracle.run_analysis(ds, selection=sel, outputs=True)
    assert np.array_equal(m2[0], mo[0, [5, 2]])


# --------------------------------------------------------------------------- F3 (float)
def test_f32_oracle_exact_cases():
    """The float instantiation (PAPER.md L172 'double variables to float variables') on data
    that float represents exactly: SPEC's worked example, identity terms, brute force."""
    g = GOLD["run_analysis"]
    ds = make_dataset(g["catalogue_size"],
                      [{"records": e["records"], "fin": [golden_value(v) for v in e["fin"]]}
                       for e in g["elts"]],
                      [{"elts": L["elts"], "terms": L["terms"]} for L in g["layers"]],
                      g["trials"])
    assert oracle.run_analysis(ds, precision=32).tolist() == g["expected_ylt"]
    cat, elts, fin, occ, agg = list(_exhaustive_cases())[0]
    trials = [list(t) for k in range(4) for t in itertools.product(range(1, cat + 1), repeat=k)]
    ds = make_dataset(cat, [{"records": sorted(e.items()), "fin": f} for e, f in zip(elts, fin)],
                      [{"elts": list(range(len(elts))), "terms": (*occ, *agg)}], trials)
    y32 = oracle.run_analysis(ds, precision=32)[0]
    for t, ev in enumerate(trials):
        assert y32[t] == trial_exact(ev, elts, fin, occ, agg)


def test_f32_separate_rounding():
    """Float line 9 = numpy float32 IEEE ops (separately rounded): catches contraction and any
    silent promotion to double inside the float instantiation."""
    rng = np.random.default_rng(78)
    x = rng.uniform(1e3, 1e8, 5000).astype(np.float32)
    r = rng.uniform(0.8, 1.25, 5000).astype(np.float32)
    t = (x * r * rng.uniform(0, 1, 5000).astype(np.float32)).astype(np.float32)
    for xi, ri, ti in zip(x, r, t):
        want = np.float32(np.float32(xi * ri) - ti)
        want = np.float32(0) if want < 0 else want
        assert oracle.apply_financial_terms_f32(float(xi), float(ri), float(ti), math.inf) == want


def _f32_accumulation_dataset():
    """Float-exact inputs whose float and double accumulations differ: 2^24 + 1 is not a float
    (it rounds to 2^24, ties to even).  Trial 0 = [1, 2, 2]: event 1's ELT sum 2^24 + 1 (lines
    11-13); trial 1 = [3, 4, 4]: exact per-event losses 2^24, 1, 1 whose running sum S (line 19)
    passes 2^24 + 1.  Identity terms, so lr = S."""
    big = float(2 ** 24)
    elts = [{"records": [(1, big), (2, 1.0), (3, big)], "fin": (1.0, 0.0, math.inf)},
            {"records": [(1, 1.0), (2, 1.0), (4, 1.0)], "fin": (1.0, 0.0, math.inf)}]
    layers = [{"elts": [0, 1], "terms": (0.0, math.inf, 0.0, math.inf)}]
    return make_dataset(8, elts, layers, [[1, 2, 2], [3, 4, 4]])


def test_f32_accumulates_in_float():
    """F3 accumulation precision: the expected values are computed with numpy float32 IEEE ops,
    the same sequence as Alg. 1 lines 11-28 in float; an instantiation that
    silently accumulated the ELT sum or S in double would give the fp64 values instead."""
    f = np.float32
    ds = _f32_accumulation_dataset()
    # trial 0: lo_1 = f(2^24) + f(1) = 2^24 (rounded), lo_2 = 2; S: 2^24, 2^24 + 2, 2^24 + 4
    lo = [f(f(f(0) + f(2 ** 24)) + f(1)), f(f(f(0) + f(1)) + f(1)), f(f(f(0) + f(1)) + f(1))]
    S, lr, prev = f(0), f(0), f(0)
    for x in lo:
        S = f(S + x)
        lr = f(lr + f(S - prev))
        prev = S
    want0 = float(lr)
    # trial 1: per-event losses 2^24, 1, 1 (exact); S rounds at 2^24 + 1 -> 2^24, twice
    S = f(0)
    for x in (f(2 ** 24), f(1), f(1)):
        S = f(S + x)
    want1 = float(S)
    y32 = oracle.run_analysis(ds, precision=32)[0]
    y64 = oracle.run_analysis(ds)[0]
    assert want0 == 2 ** 24 + 4 and want1 == 2 ** 24
    assert y32.tolist() == [want0, want1]
    assert y64.tolist() == [2 ** 24 + 5, 2 ** 24 + 2]  # double accumulation: different


def test_f32_within_rounding_bound_of_f64():
    """fp32 vs fp64 on generated data: |y32 - y64| within the absolute rounding bound of float
    arithmetic over the trial, c (k + E + 2) u32 (S + AggR), u32 = 2^-24 (input rounding
    included); SPEC.md L283's 1e-4 relative bar is reported, not asserted, because S - AggR
    cancels (F3)."""
    ds = datagen.generate(datagen.PRESETS["tiny"].replace(n_trials=1000, seed=3))
    y64 = oracle.run_analysis(ds)[0]
    y32 = oracle.run_analysis(ds, precision=32)[0]
    occR, occL, aggR, aggL = ds.layer_terms[0]
    S = oracle.run_analysis(ds, precision=64, trial_offsets=ds.trial_offsets)[0]  # noqa: F841
    u32 = 2.0 ** -24
    bound = 8 * (10 + 2 + 2) * u32 * (aggR + aggL + float(np.max(ds.rec_losses)) * 2 * 10)
    assert np.all(np.abs(y32 - y64) <= bound)
    assert np.mean(np.abs(y32 - y64) <= 1e-4 * np.abs(y64) + 1e-300) > 0.5


# --------------------------------------------------------------------------- portfolio scope
def test_portfolio_row_pins():
    """Portfolio-scope losses (per-trial sum over layers): one layer gives the
    layer's row unchanged; small dyadic YLTs sum exactly (checked in exact rationals); the sum
    runs left to right in layer order (1e16 + 1 + 1 rounds to 1e16, 1 + 1 + 1e16 does not)."""
    from fractions import Fraction
    rng = np.random.default_rng(11)
    row = rng.lognormal(10, 2, 257)
    assert np.array_equal(oracle.portfolio_row(row[None, :]), row)
    for L in (2, 3, 8):
        y = rng.integers(0, 1 << 30, size=(L, 100)).astype(float) / 1024.0
        got = oracle.portfolio_row(y)
        for t in range(100):
            assert Fraction(got[t]) == sum(Fraction(v) for v in y[:, t])
    y = np.array([[1e16, 1.0], [1.0, 1.0], [1.0, 1e16]])
    got = oracle.portfolio_row(y)
    assert got[0] == 1e16 and got[1] == 1.0000000000000002e16
    # monotone: adding a layer never lowers a trial's portfolio loss (all entries >= 0)
    y = rng.lognormal(5, 3, (4, 50))
    assert (oracle.portfolio_row(y) >= oracle.portfolio_row(y[:3])).all()


# --------------------------------------------------------------------------- F4 EP curves
def test_ep_curve_pins():
    """Exceedance-probability curve (F4, reading R15): SPEC's 1..100 row gives 100, 99, ..., 1
    and its PML(0.99) = 99 sits at rank n - ceil(p n); on random rows with ties
    the curve is non-increasing, a permutation of the row (numpy's sort, an independent library
    routine), every entry i has at least i + 1 values >= it and at most i values > it (brute
    force), and the nearest-rank PML of every return period is a point on it."""
    v = np.arange(1.0, 101.0)
    rng = np.random.default_rng(15)
    c = oracle.ep_curve(rng.permutation(v))
    assert c.tolist() == list(np.arange(100.0, 0.0, -1.0))
    assert c[100 - math.ceil(0.99 * 100)] == oracle.metrics(v, [0.99])[0][0] == 99.0
    p = [1 - 1 / rp for rp in (10, 25, 50, 100, 250, 500, 1000)]
    for trial in range(200):
        n = int(rng.integers(1, 400))
        row = np.round(rng.lognormal(3, 2, n), 1 if trial % 2 else 8)  # ties when rounded
        c = oracle.ep_curve(row)
        assert (np.diff(c) <= 0).all()
        assert np.array_equal(np.sort(row)[::-1], c)
        if n <= 60:
            for i in range(n):
                assert (row >= c[i]).sum() >= i + 1 and (row > c[i]).sum() <= i
        pml = oracle.metrics(row, p)[0]
        for pi, q in zip(p, pml):
            assert c[n - math.ceil(pi * n)] == q
    assert oracle.ep_curve(np.array([7.5])).tolist() == [7.5]
    with pytest.raises(ValueError):
        oracle.ep_curve(np.array([]))
