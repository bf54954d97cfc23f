"""Test helpers: small explicit datasets and exact (rational) reference formulations.

The exact formulations here are NOT a retyping of Algorithm 1.  They use the textbook
characterisation of an excess-of-loss layer (cover "up to a specified limit with an
optional retention") as the length of an interval intersection:

    xl(x; R, L)        = |[0, x] cap [R, R + L]|           (what a layer R xs L pays on loss x)
    paid(a, b; R, L)   = |[a, b] cap [R, R + L]|           (what an aggregate layer pays for the
                                                            slice of cumulative loss from a to b)

An occurrence moves the trial's cumulative loss from S_{d-1} to S_d; the aggregate layer pays
exactly the part of that move that falls inside [AggR, AggR + AggL] ("erosion" of the layer).
Algorithm 1 instead clamps every prefix sum and differences them (lines 18-26); the two agree
in exact arithmetic, which is the point of using them as a pin.
"""
from __future__ import annotations

import math
import types
from fractions import Fraction
from typing import Dict, List, Sequence

import numpy as np

INF = math.inf


def F(x) -> Fraction:
    return Fraction(x)


def seg(a, b, lo, hi):
    """|[a, b] cap [lo, hi]| with hi possibly +inf (exact rationals)."""
    top = b if hi == INF else min(b, hi)
    return max(Fraction(0), top - max(a, lo))


def xl(x, ret, lim):
    """Layer 'lim xs ret' applied to a single loss x >= 0."""
    return seg(Fraction(0), x, ret, INF if lim == INF else ret + lim)


def trial_exact(events: Sequence[int], elts: List[Dict[int, Fraction]], fin, occ, agg):
    """Exact trial loss by the erosion formulation (see module docstring).
    fin[j] = (rate, ret, lim); occ = (OccR, OccL); agg = (AggR, AggL)."""
    agg_hi = INF if agg[1] == INF else F(agg[0]) + F(agg[1])
    s_prev = Fraction(0)
    total = Fraction(0)
    for e in events:
        lo = Fraction(0)
        for j, table in enumerate(elts):
            rate, ret, lim = fin[j]
            lo += xl(F(table.get(e, 0)) * F(rate), F(ret), lim if lim == INF else F(lim))
        oc = xl(lo, F(occ[0]), occ[1] if occ[1] == INF else F(occ[1]))
        s = s_prev + oc
        total += seg(s_prev, s, F(agg[0]), agg_hi)
        s_prev = s
    return total


def trial_S_exact(events, elts, fin, occ):
    s = Fraction(0)
    for e in events:
        lo = Fraction(0)
        for j, table in enumerate(elts):
            rate, ret, lim = fin[j]
            lo += xl(F(table.get(e, 0)) * F(rate), F(ret), lim if lim == INF else F(lim))
        s += xl(lo, F(occ[0]), occ[1] if occ[1] == INF else F(occ[1]))
    return s


def make_dataset(catalogue_size: int, elts: List[dict], layers: List[dict],
                 trials: List[Sequence[int]]):
    """elts: [{"records": [(id, loss), ...], "fin": (rate, ret, lim)}];
    layers: [{"elts": [j, ...], "terms": (OccR, OccL, AggR, AggL)}]; trials: [[id, ...]]."""
    rec_off = [0]
    ids, losses, fin = [], [], []
    for e in elts:
        for i, l in e["records"]:
            ids.append(i); losses.append(l)
        rec_off.append(len(ids))
        fin.append([float(v) for v in e["fin"]])
    eo, ei, lt = [0], [], []
    for L in layers:
        ei.extend(L["elts"]); eo.append(len(ei)); lt.append([float(v) for v in L["terms"]])
    to = [0]
    ev = []
    for t in trials:
        ev.extend(t); to.append(len(ev))
    return types.SimpleNamespace(
        catalogue_size=catalogue_size, n_layers=len(layers), n_trials=len(trials),
        rec_offsets=np.array(rec_off, dtype=np.uint64),
        rec_event_ids=np.array(ids, dtype=np.uint32),
        rec_losses=np.array(losses, dtype=np.float64),
        fin=np.array(fin, dtype=np.float64).reshape(-1, 3),
        layer_terms=np.array(lt, dtype=np.float64).reshape(-1, 4),
        elt_offsets=np.array(eo, dtype=np.uint32),
        elt_index=np.array(ei, dtype=np.uint32),
        trial_offsets=np.array(to, dtype=np.uint64),
        events=np.array(ev, dtype=np.uint32))


def elt_dicts(ds, layer: int):
    """Per-ELT {event: loss} dicts of one layer, in layer order, plus its fin terms."""
    out, fin = [], []
    for c in range(int(ds.elt_offsets[layer]), int(ds.elt_offsets[layer + 1])):
        j = int(ds.elt_index[c])
        a, b = int(ds.rec_offsets[j]), int(ds.rec_offsets[j + 1])
        out.append({int(i): float(l) for i, l in zip(ds.rec_event_ids[a:b], ds.rec_losses[a:b])})
        fin.append(tuple(float(v) for v in ds.fin[j]))
    return out, fin


def trial_events(ds, t: int):
    return [int(e) for e in ds.events[int(ds.trial_offsets[t] - ds.trial_offsets[0]):
                                      int(ds.trial_offsets[t + 1] - ds.trial_offsets[0])]]


def golden_value(v):
    return INF if v == "inf" else v
