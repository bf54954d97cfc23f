"""GPU parity at BASELINE.json configs[1] and configs[2] sizes, every YLT entry, plus the kernel
selection, the multi-process sharded path and the C-ABI error contracts.

Every entry of the YLT is compared with the oracle (bit-identical, -0 == +0), and PML/TVaR of the
GPU YLT with oracle.metrics of the oracle YLT (PML exact, TVaR within 1e-9; PAPER.md L32, L110-L112;
SURVEY.md T2).  Each full-size case runs twice on one context: the first run probes the YET and
takes the bitmap / length-check path, the second launches the kernel the previous run's verdicts
select -- the steady-state kernel bench.py times.
"""
import json
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import datagen
import oracle
from tests._util import make_dataset

torch = pytest.importorskip("torch")
from paper_1308_2572_b200 import ara  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P_RP = [1 - 1 / rp for rp in (10, 25, 50, 100, 250, 500, 1000)]
THREADS = max(1, len(os.sched_getaffinity(0)))


def to_dev(a, kind):
    if kind == "u64":
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).to(DEV).view(torch.uint64)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to(DEV).view(torch.uint32)


def ctx_for(ds):
    ctx = ara.Context(0, torch.cuda.current_stream(torch.device(DEV)))
    ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses, ds.fin)
    ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
    return ctx


def check_every_entry(got, want):
    assert got.shape == want.shape
    bad = np.flatnonzero(got.ravel() != want.ravel())
    assert bad.size == 0, (f"{bad.size} of {got.size} YLT entries differ; first {bad[:5]}: gpu "
                           f"{got.ravel()[bad[:5]]} oracle {want.ravel()[bad[:5]]}")


def check_metrics(ctx, d_row, want_row):
    pml, tvar = ctx.ara_metrics(d_row, P_RP)
    opml, otvar = oracle.metrics(want_row, P_RP)
    assert np.array_equal(pml, opml), (pml, opml)
    assert np.allclose(tvar, otvar, rtol=1e-9, atol=0), (tvar, otvar)


@pytest.mark.parametrize("config", ["medium", "headline"])
def test_full_size_every_entry_twice(config):
    """configs[1] (100,000 x 1,000) and the headline (1,000,000 x 1,000): every YLT entry and
    PML/TVaR at the seven return periods, on two consecutive runs of one context."""
    ds = datagen.generate(datagen.PRESETS[config])
    want = oracle.run_analysis(ds, n_threads=THREADS)
    ctx = ctx_for(ds)
    d_off, d_ev = to_dev(ds.trial_offsets, "u64"), to_dev(ds.events, "u32")
    kernels = []
    for _ in range(2):
        ylt = torch.full((ds.n_layers, ds.n_trials), math.nan, dtype=torch.float64, device=DEV)
        ctx.ara_run(d_off, d_ev, ylt, flags=ara.ARA_RUN_SYNC)
        check_every_entry(ylt.cpu().numpy(), want)
        check_metrics(ctx, ylt[0], want[0])
        kernels.append(ctx.ara_get_info().last_kernel.decode())
        curve = torch.empty(ds.n_trials, dtype=torch.float64, device=DEV)  # F4 AEP curve
        ctx.ara_ep_curve(ylt[0], curve)
        check_every_entry(curve.cpu().numpy(), oracle.ep_curve(want[0]))
        torch.cuda.synchronize()
    # 16 ELTs, every event in the store (h = 1): the second run launches the plain row-by-id
    # instantiation of the pair scan (the kernel bench.py times)
    assert kernels[1] == "pair_scan_kernel<2, 2, 3, 1, 0, 1>", kernels
    ctx.close()


def _adversarial(n_elts: int, scale: float = 1.0):
    rng = np.random.default_rng(11)
    cat = 64
    elts = []
    for j in range(n_elts):
        ids = rng.choice(np.arange(1, cat + 1), 40, replace=False)
        ls = rng.uniform(0.1, 1e6, 40) * (10.0 ** rng.integers(-3, 4, 40)) * scale
        fin = (1.0 + rng.uniform(-0.3, 0.3), float(rng.uniform(0, 1e4)) * scale,
               math.inf if j % 2 else float(rng.uniform(1e4, 1e6)) * scale)
        if j == 3:
            fin = (fin[0], 0.0, 0.0)  # a zero limit: the column pays nothing
        elts.append({"records": list(zip(ids.tolist(), ls.tolist())), "fin": fin})
    trials = [list(rng.integers(1, cat + 1, rng.integers(0, 60))) for _ in range(400)]
    trials += [[3] * 50, [], [1], list(range(1, cat + 1))]
    return cat, elts, trials


@pytest.mark.parametrize("n_elts", [9, 16])
def test_adversarial_pair_scan(n_elts):
    """The cancellation cases (AggR at / next to exact trial sums, AggR + AggL = S, OccR equal to
    an event's combined loss, zero and infinite limits) through the exactly scaled pair scan:
    bit-identical to the unscaled oracle."""
    cat, elts, trials = _adversarial(n_elts)
    all_elts = list(range(n_elts))
    ident = make_dataset(cat, elts, [{"elts": all_elts, "terms": (0, math.inf, 0, math.inf)}],
                         trials)
    S = oracle.run_analysis(ident)[0]
    single = oracle.run_analysis(make_dataset(
        cat, elts, [{"elts": all_elts, "terms": (0, math.inf, 0, math.inf)}],
        [[e] for e in range(1, cat + 1)]))[0]
    cases = []
    for t in (0, 5, 17, 123):
        cases += [(0.0, math.inf, float(S[t]), math.inf), (0.0, math.inf, float(S[t]), 1.0),
                  (0.0, math.inf, float(np.nextafter(S[t], 0)), math.inf),
                  (0.0, math.inf, float(S[t]) / 2, float(S[t]) / 2)]
    cases += [(float(single[2]), math.inf, 0.0, math.inf), (0.0, 0.0, 0.0, math.inf),
              (10.0, 1e5, 0.0, 0.0), (1e9, math.inf, 0.0, math.inf)]
    for c in cases:  # one layer per case: each run takes the single-layer pair scan
        ds = make_dataset(cat, elts, [{"elts": all_elts, "terms": c}], trials)
        ctx = ctx_for(ds)
        ylt = torch.empty((1, ds.n_trials), dtype=torch.float64, device=DEV)
        ctx.ara_run(to_dev(ds.trial_offsets, "u64"), to_dev(ds.events, "u32"), ylt,
                    flags=ara.ARA_RUN_SYNC)
        check_every_entry(ylt.cpu().numpy(), oracle.run_analysis(ds))
        assert ctx.ara_get_info().last_kernel.decode().startswith("pair_scan_kernel<2, 2,")
        ctx.close()


@pytest.mark.parametrize("scale,pair", [(2.0 ** 900, True), (2.0 ** 960, False)])
def test_scaled_path_guard(scale, pair):
    """Inputs whose magnitudes could overflow the scaled intermediates (>= 2^960) run the
    compare-select kernel; both paths are bit-identical to the oracle."""
    cat, elts, trials = _adversarial(16, scale)
    ds = make_dataset(cat, elts, [{"elts": list(range(16)),
                                   "terms": (1e4 * scale, math.inf, 1e5 * scale, 1e9 * scale)}],
                      trials)
    ctx = ctx_for(ds)
    ylt = torch.empty((1, ds.n_trials), dtype=torch.float64, device=DEV)
    ctx.ara_run(to_dev(ds.trial_offsets, "u64"), to_dev(ds.events, "u32"), ylt,
                flags=ara.ARA_RUN_SYNC)
    check_every_entry(ylt.cpu().numpy(), oracle.run_analysis(ds))
    assert ctx.ara_get_info().last_kernel.decode().startswith(
        "pair_scan_kernel" if pair else "scan_kernel")
    ctx.close()


def test_validate_offsets_end_below_start():
    """ARA_RUN_VALIDATE with offsets[n] < offsets[0] (interior order irrelevant) fails with
    ARA_ERR_VALIDATION before any kernel reads ids, and the context stays usable."""
    ds = datagen.generate(datagen.PRESETS["tiny"])
    ctx = ctx_for(ds)
    bad = ds.trial_offsets.copy()
    bad[0], bad[-1] = bad[-1], 0
    ylt = torch.empty((1, ds.n_trials), dtype=torch.float64, device=DEV)
    with pytest.raises(ara.AraError) as e:
        ctx.ara_run(to_dev(bad, "u64"), to_dev(ds.events, "u32"), ylt, flags=ara.ARA_RUN_VALIDATE)
    assert e.value.status_name == "ARA_ERR_VALIDATION"
    ctx.ara_run(to_dev(ds.trial_offsets, "u64"), to_dev(ds.events, "u32"), ylt,
                flags=ara.ARA_RUN_SYNC | ara.ARA_RUN_VALIDATE)
    check_every_entry(ylt.cpu().numpy(), oracle.run_analysis(ds))
    ctx.close()


@pytest.mark.parametrize("flags", [0, ara.ARA_RUN_VALIDATE])
def test_run_host_error_writes_nothing(flags):
    """ara_run_host with an out-of-range event id returns ARA_ERR_RANGE and leaves the caller's
    YLT untouched (ara.h: on failure nothing is written to caller outputs)."""
    ds = datagen.generate(datagen.PRESETS["tiny"])
    ctx = ctx_for(ds)
    ev = ds.events.copy()
    ev[len(ev) // 2] = ds.catalogue_size + 5
    h = np.full((1, ds.n_trials), -3.0)
    with pytest.raises(ara.AraError) as e:
        ctx.ara_run_host(ds.trial_offsets, ev, h, flags=flags)
    assert e.value.status_name == "ARA_ERR_RANGE"
    assert (h == -3.0).all()
    ctx.ara_run_host(ds.trial_offsets, ds.events, h, flags=flags)  # still usable
    check_every_entry(h, oracle.run_analysis(ds))
    ctx.close()


def test_two_ranks_sharded_path():
    """The multi-GPU path of bench.py with 2 processes sharing this GPU (gloo): each rank scans
    its trial slice through libara, the slices are all-gathered (dist.gather_ylt) and PML/TVaR
    computed (ara_metrics_rows) on rank 0, which scans fewer trials to make up for it; rank 0
    compares the gathered YLT of the last timed step with the single-process oracle over the
    whole workload, every entry."""
    env = dict(os.environ, ARA_BENCH_SAME_DEVICE="1", MASTER_ADDR="127.0.0.1")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
         "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(ROOT, "bench.py"),
         "--gpus", "2", "--config", "medium", "--steps", "3", "--warmup", "3", "--no-e2e"],
        capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    # rank 0 computes PML/TVaR alone and scans fewer trials (dist.partition_rank0_offload)
    by_rank = d["config"]["trials_by_rank"]
    assert d["config"]["trials"] == 100_000 and sum(by_rank) == 100_000
    assert by_rank[0] == d["config"]["trials_per_gpu"] and by_rank[0] <= 50_000 <= by_rank[1]
    assert d["config"]["metrics_on"].startswith("rank 0")
    p = d["parity"]
    assert p["pass"] and p["ylt_mismatches"] == 0 and p["ylt_n"] == 100_000 and p["pml_exact"]


def test_nccl_collectives_single_rank():
    """dist.py's NCCL branches, which no multi-GPU box has run yet: one rank under torchrun with
    an NCCL process group on this GPU (NCCL refuses two ranks on one device) broadcasts the
    inputs, scans its slice through libara, all-gathers the YLT (all_gather_into_tensor) and
    computes PML/TVaR both from the gathered row and by the all-reduced sharded radix select;
    every YLT entry and PML equal the oracle's, TVaR within 1e-9 (tests/_nccl_rank.py)."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
         "--master-addr", "127.0.0.1", "--master-port", "29563",
         os.path.join(ROOT, "tests", "_nccl_rank.py")],
        capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    d = json.loads(lines[-1])
    assert d["backend"] == "nccl" and d["world"] == 1
    assert d["20000"]["mismatches"] == 0 and d["20001"]["mismatches"] == 0


def test_oep_curve_from_max_occ():
    """F4 OEP: the exceedance curve of the per-trial maximum occurrence losses (ara_run_outputs
    max_occ, reading R13) equals the oracle's sorted max_occ row, entry by entry; the AEP curve of
    the same run equals the oracle's sorted YLT."""
    ds = datagen.generate(datagen.PRESETS["medium"].replace(n_trials=20_000))
    want, mo, _ = oracle.run_analysis(ds, n_threads=THREADS, outputs=True)
    ctx = ctx_for(ds)
    ylt = torch.empty((1, ds.n_trials), dtype=torch.float64, device=DEV)
    d_mo = torch.empty((1, ds.n_trials), dtype=torch.float64, device=DEV)
    ctx.ara_run_outputs(to_dev(ds.trial_offsets, "u64"), to_dev(ds.events, "u32"), ylt,
                        d_max_occ=d_mo, flags=ara.ARA_RUN_SYNC)
    oep = torch.empty(ds.n_trials, dtype=torch.float64, device=DEV)
    aep = torch.empty(ds.n_trials, dtype=torch.float64, device=DEV)
    ctx.ara_ep_curve(d_mo[0], oep)
    ctx.ara_ep_curve(ylt[0], aep)
    check_every_entry(oep.cpu().numpy(), oracle.ep_curve(mo[0]))
    check_every_entry(aep.cpu().numpy(), oracle.ep_curve(want[0]))
    # every PML is a point of the AEP curve: PML(p) = curve[n - ceil(p n)]
    pml, _ = ctx.ara_metrics(ylt[0], P_RP)
    c = aep.cpu().numpy()
    assert [c[ds.n_trials - math.ceil(p * ds.n_trials)] for p in P_RP] == pml.tolist()
    ctx.close()


def test_ep_curve_edges():
    """n = 1, ties, -0 -> +0; empty rows and overlapping buffers are rejected."""
    ds = datagen.generate(datagen.PRESETS["tiny"])
    ctx = ctx_for(ds)
    for row in ([5.0], [3.0, 3.0, -0.0, 7.0, 3.0, 0.0], list(np.arange(1.0, 1001.0))):
        d = torch.tensor(row, dtype=torch.float64, device=DEV)
        out = torch.empty_like(d)
        ctx.ara_ep_curve(d, out)
        got = out.cpu().numpy()
        assert got.tolist() == sorted([abs(x) if x == 0 else x for x in row], reverse=True)
        assert not np.signbit(got).any()
    with pytest.raises(ara.AraError) as e:
        ctx.ara_ep_curve(torch.empty(0, dtype=torch.float64, device=DEV),
                         torch.empty(0, dtype=torch.float64, device=DEV))
    assert e.value.status_name == "ARA_ERR_EMPTY"
    buf = torch.zeros(10, dtype=torch.float64, device=DEV)
    with pytest.raises(ara.AraError) as e:
        ctx.ara_ep_curve(buf[:6], buf[4:])
    assert e.value.status_name == "ARA_ERR_ARG"
    ctx.close()


def test_f32_accumulates_in_float_on_gpu():
    """F3 on the GPU: the float-accumulation pin dataset (tests/test_oracle_pins.py) gives the
    float oracle's values, which differ from double accumulation."""
    from tests.test_oracle_pins import _f32_accumulation_dataset
    ds = _f32_accumulation_dataset()
    ctx = ara.Context(0, torch.cuda.current_stream(torch.device(DEV)))
    ctx.ara_set_precision(32)
    ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses, ds.fin)
    ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
    ylt = torch.empty((1, 2), dtype=torch.float64, device=DEV)
    ctx.ara_run(to_dev(ds.trial_offsets, "u64"), to_dev(ds.events, "u32"), ylt,
                flags=ara.ARA_RUN_SYNC)
    assert ylt.cpu().numpy()[0].tolist() == [2.0 ** 24 + 4, 2.0 ** 24]
    ctx.close()
