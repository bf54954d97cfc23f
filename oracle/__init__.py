"""ctypes wrapper around ``oracle/liboracle.so`` -- the plain fp64 CPU oracle.

TEST INFRASTRUCTURE ONLY.  Importable from ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``; never from the product package
``paper_1308_2572_b200``.  It shares no code with the CUDA path (see ``oracle/oracle.c`` for the
paper citations and the readings R1-R12 of DESIGN.md).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_INC = os.path.join(_HERE, "alg1.inc")
_LIB = os.path.join(_HERE, "liboracle.so")

# -ffp-contract=off: products and differences are rounded separately (no FMA), as the
# oracle's arithmetic requires (reading R7).
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(_INC)):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lpthread", "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        d, u32, u64, i64, p = (ctypes.c_double, ctypes.c_uint32, ctypes.c_uint64,
                               ctypes.c_int64, ctypes.c_void_p)
        L.oracle_apply_financial_terms.argtypes = [d, d, d, d]
        L.oracle_apply_financial_terms.restype = d
        L.oracle_apply_occurrence_terms.argtypes = [d, d, d]
        L.oracle_apply_occurrence_terms.restype = d
        L.oracle_apply_aggregate_terms.argtypes = [p, u64, d, d, p, p]
        L.oracle_apply_aggregate_terms.restype = None
        L.oracle_build_dat.argtypes = [u32, u64, p, p, p]
        L.oracle_build_dat.restype = i64
        L.oracle_run_analysis.argtypes = [u32, u32, p, p, p, p, u32, p, p, p, u64, p, p,
                                          u64, p, p, ctypes.c_int]
        L.oracle_run_analysis.restype = ctypes.c_int
        L.oracle_run_analysis_ex.argtypes = [u32, u32, p, p, p, p, u32, p, p, p, u64, p, p,
                                             u64, p, p, p, p, ctypes.c_int]
        L.oracle_run_analysis_ex.restype = ctypes.c_int
        L.oracle_run_analysis_f32.argtypes = L.oracle_run_analysis_ex.argtypes
        L.oracle_run_analysis_f32.restype = ctypes.c_int
        f = ctypes.c_float
        L.oracle_apply_financial_terms_f32.argtypes = [f, f, f, f]
        L.oracle_apply_financial_terms_f32.restype = f
        L.oracle_apply_occurrence_terms_f32.argtypes = [f, f, f]
        L.oracle_apply_occurrence_terms_f32.restype = f
        L.oracle_metrics.argtypes = [p, u64, u32, p, p, p]
        L.oracle_metrics.restype = ctypes.c_int
        L.oracle_ep_curve.argtypes = [p, u64, p]
        L.oracle_ep_curve.restype = ctypes.c_int
        L.oracle_portfolio_row.argtypes = [p, u32, u64, u64, p]
        L.oracle_portfolio_row.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def apply_financial_terms(x: float, rate: float, retention: float, limit: float) -> float:
    """Alg. 1 line 9 under reading R1."""
    return lib().oracle_apply_financial_terms(x, rate, retention, limit)


def apply_financial_terms_f32(x, rate, retention, limit) -> float:
    """Line 9 in float arithmetic (F3)."""
    return lib().oracle_apply_financial_terms_f32(x, rate, retention, limit)


def apply_occurrence_terms(lo: float, occ_retention: float, occ_limit: float) -> float:
    """Alg. 1 line 16."""
    return lib().oracle_apply_occurrence_terms(lo, occ_retention, occ_limit)


def apply_aggregate_terms(lo: Sequence[float], agg_retention: float, agg_limit: float):
    """Alg. 1 lines 18-26: per-event incremental aggregate losses."""
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    k = lo.shape[0]
    cum = np.empty(max(k, 1)); inc = np.empty(max(k, 1))
    lib().oracle_apply_aggregate_terms(_ptr(lo), k, agg_retention, agg_limit, _ptr(cum),
                                       _ptr(inc))
    return inc[:k].copy()


def build_dat(catalogue_size: int, event_ids, losses) -> np.ndarray:
    """Direct access table of one ELT: length C+1, absent events 0."""
    ids = np.ascontiguousarray(event_ids, dtype=np.uint32)
    ls = np.ascontiguousarray(losses, dtype=np.float64)
    dat = np.empty(catalogue_size + 1, dtype=np.float64)
    bad = lib().oracle_build_dat(catalogue_size, ids.shape[0], _ptr(ids), _ptr(ls), _ptr(dat))
    if bad:
        raise ValueError(f"record {bad - 1}: event id {int(ids[bad - 1])} outside [1, "
                         f"{catalogue_size}]")
    return dat


def run_analysis(ds, selection: Optional[np.ndarray] = None, n_threads: int = 1,
                 trial_offsets=None, events=None, outputs: bool = False, precision: int = 64):
    """YLT[n_layers][n] of Algorithm 1.

    ``ds`` carries numpy arrays: catalogue_size, rec_offsets, rec_event_ids, rec_losses,
    fin[n_elts,3] (rate, retention, limit), layer_terms[n_layers,4] (OccR, OccL, AggR, AggL),
    elt_offsets, elt_index, trial_offsets, events.  ``selection``: optional trial indices.
    """
    c = lambda a, t: np.ascontiguousarray(a, dtype=t)  # noqa: E731
    rec_off = c(ds.rec_offsets, np.uint64)
    rec_ids = c(ds.rec_event_ids, np.uint32)
    rec_ls = c(ds.rec_losses, np.float64)
    fin = c(ds.fin, np.float64)
    lt = c(ds.layer_terms, np.float64)
    eo = c(ds.elt_offsets, np.uint32)
    ei = c(ds.elt_index, np.uint32)
    to = c(ds.trial_offsets if trial_offsets is None else trial_offsets, np.uint64)
    ev = c(ds.events if events is None else events, np.uint32)
    n_layers = eo.shape[0] - 1
    n_trials = to.shape[0] - 1
    sel = None if selection is None else c(selection, np.uint64)
    n_out = n_trials if sel is None else sel.shape[0]
    ylt = np.zeros((n_layers, n_out), dtype=np.float64)
    n_ev = int(to[-1] - to[0]) if to.size else 0
    mo = np.zeros((n_layers, n_out)) if outputs else None
    inc = np.zeros((n_layers, max(n_ev, 1))) if outputs else None
    if n_layers == 0 or n_out == 0:
        return (ylt, mo, inc[:, :n_ev]) if outputs else ylt
    fn = lib().oracle_run_analysis_ex if precision == 64 else lib().oracle_run_analysis_f32
    if precision not in (32, 64):
        raise ValueError("precision must be 32 or 64")
    st = fn(
        int(ds.catalogue_size), rec_off.shape[0] - 1, _ptr(rec_off), _ptr(rec_ids),
        _ptr(rec_ls), _ptr(fin), n_layers, _ptr(lt), _ptr(eo),
        _ptr(ei) if ei.size else None, n_trials, _ptr(to),
        _ptr(ev) if ev.size else None, 0 if sel is None else sel.shape[0],
        None if sel is None else _ptr(sel), _ptr(ylt), _ptr(mo) if outputs else None,
        _ptr(inc) if outputs else None, int(n_threads))
    if st == -1:
        raise MemoryError("oracle: out of memory")
    if st == -3:
        raise ValueError("oracle: trial event id outside [1, catalogue_size]")
    if st < -1:
        raise ValueError(f"oracle: ELT record {-st - 2} has an invalid event id")
    return (ylt, mo, inc[:, :n_ev]) if outputs else ylt


def portfolio_row(ylt) -> np.ndarray:
    """Portfolio-scope trial losses: per trial, the sum over layers in layer order, left to
    right from +0."""
    y = np.ascontiguousarray(ylt, dtype=np.float64)
    if y.ndim == 1:
        y = y[None, :]
    out = np.empty(y.shape[1])
    lib().oracle_portfolio_row(_ptr(y), y.shape[0], y.shape[1], y.shape[1], _ptr(out))
    return out


def metrics(ylt_row, p: Sequence[float]):
    """(PML, TVaR) arrays at probabilities p (reading R11)."""
    v = np.ascontiguousarray(ylt_row, dtype=np.float64)
    pp = np.ascontiguousarray(p, dtype=np.float64)
    pml = np.empty(pp.shape[0]); tvar = np.empty(pp.shape[0])
    st = lib().oracle_metrics(_ptr(v), v.shape[0], pp.shape[0], _ptr(pp), _ptr(pml),
                              _ptr(tvar))
    if st == -1:
        raise ValueError("oracle: empty YLT")
    if st == -2:
        raise ValueError("oracle: p outside (0, 1)")
    if st:
        raise MemoryError("oracle: out of memory")
    return pml, tvar


def ep_curve(row) -> np.ndarray:
    """Exceedance-probability curve (F4, reading R15): the row sorted from the largest value
    down; entry i has empirical exceedance probability (i+1)/n.  AEP from a YLT row, OEP from
    the per-trial maximum occurrence losses."""
    v = np.ascontiguousarray(row, dtype=np.float64)
    out = np.empty(v.shape[0])
    if lib().oracle_ep_curve(_ptr(v), v.shape[0], _ptr(out)) == -1:
        raise ValueError("oracle: empty row")
    return out
