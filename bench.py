#!/usr/bin/env python3
"""Benchmark of the hot path: YET trial-events/s (BASELINE.json metric) on 1..N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config headline] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N           (N > 1, one process per GPU)

A step is one pass of the whole hot path over one batch: every rank
scans its contiguous trial slice of the YET (ara_run: A2-A8, device-resident inputs), the YLT
slices are all-gathered over NCCL (N > 1), and PML/TVaR at the return periods are computed
(ara_metrics: A9).  The ELT store build (A1, ara_set_layers) is setup and not timed (it is the
paper's preprocessing stage).  Strong scaling by default: the configured workload
(1M trials at the headline) is split over the ranks, as the paper decomposed one fixed workload
over its GPUs; ``--scaling weak`` gives every rank the whole workload's
trial count instead.  Inputs are synthetic (datagen/, seed 1308) with the paper's workload shape.

Timing: W untimed warm-up steps, then K steps bracketed by barrier + synchronize, CUDA events on
the context stream, max over ranks.  The YET (4 GB at the headline) is larger than L2, so every
step streams it from HBM; the ELT rows are L2-resident by design.  `e2e` repeats the step through
the host-buffer C-ABI call (ara_run_host: pinned host YET copied in every step, YLT copied back).

Parity (rank 0, after timing): the CPU oracle (oracle/, test infrastructure) runs Algorithm 1
over every trial of the workload on the host cores; the YLT of the LAST timed step is compared
with it entry by entry, and the step's PML/TVaR with the oracle's metrics of the oracle YLT
(``parity`` in the JSON line).  The same oracle run is the ``cpu_baseline`` (N = 1).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

RETURN_PERIODS = (10, 25, 50, 100, 250, 500, 1000)
P = [1.0 - 1.0 / rp for rp in RETURN_PERIODS]
METRIC = "YET trial-events/sec at 1M×1000, 1/2/4/8 B200; % of HBM roofline"
UNIT = "trial-events/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def partition(n: int, r: int, R: int):
    """Contiguous balanced trial range of rank r."""
    from paper_1308_2572_b200.dist import shard_range
    return shard_range(n, r, R)


def workload_name(spec) -> str:
    k = f"{spec.k_min}" if spec.k_min == spec.k_max else f"{spec.k_min}-{spec.k_max}"
    return (f"{spec.name}: {spec.n_layers} layer(s), {spec.elts_per_layer} ELTs/layer x "
            f"{spec.records_per_elt} records, catalogue {spec.catalogue_size}, pool "
            f"{spec.pool_size}, {spec.n_trials} trials x {k} events, hit {spec.hit}, "
            f"seed {spec.seed}")


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def gather_ceiling():
    """Best measured rate of random 128-byte row gathers from L2 on this B200 (the scan's binding
    resource: rows are L2 hits, DRAM carries only the id stream).  From the committed
    microbenchmark (tools/microbench_rowpattern.cu): the fastest layout at any occupancy."""
    import glob
    best, src = None, None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*microbench_rowpattern*.jsonl"))):
        for line in open(path):
            d = json.loads(line)
            if "events_per_s" in d and (best is None or d["events_per_s"] > best):
                best, src = d["events_per_s"], f"{os.path.relpath(path, ROOT)}: {d['kernel']} " \
                                                 f"at grid {d['grid']}"
    return best, src


def ncu_entry(kernel: str, config: str):
    """The committed ncu counters (profiles/scan_traffic.json) of THIS kernel instantiation built
    from THESE sources (paper_1308_2572_b200.build.source_sha16) and config, else None (stale
    counters are never reported)."""
    from paper_1308_2572_b200.build import source_sha16
    path = os.path.join(ROOT, "profiles", "scan_traffic.json")
    try:
        j = json.load(open(path))
    except Exception:
        return None
    e = j.get(f"{kernel}|{source_sha16()}|{config}")
    return e if isinstance(e, dict) else None


def roofline(args, spec, ctx, info, n_ev: int, n_loc: int, scan_ms: float) -> dict:
    """Roofline of the dominant kernel (the scan), per launch on this rank.

    Binding resource: random row gathers from L2 -- every trial-event
    gathers its rows (gather_row_bytes) from the L2-resident store; `achieved` is those bytes over
    the kernel time and `peak` the best measured 128-byte row-gather rate.  The north-star HBM
    accounting (ids + E-wide rows + YLT + offsets against the copy bandwidth) is kept as the
    secondary `north_star` view: its fraction exceeds 1 because the rows are L2 hits."""
    L, E = spec.n_layers, spec.elts_per_layer
    vb = args.precision // 8
    t = scan_ms * 1e-3
    peak_hbm, peak_src = measured_peak()
    alg = n_ev * (4 + vb * E * L) + 8 * n_loc * L + 8 * (n_loc + 1)
    ns = {"bound": "hbm", "unit": "GB/s", "bytes_alg_per_launch": alg,
          "achieved": alg / t / 1e9, "peak": peak_hbm, "peak_source": peak_src,
          "frac": alg / t / 1e9 / peak_hbm,
          "bytes_model": f"n*k*(4 + {vb}*E*L) + 8*n*L + 8*(n+1): ids once, each layer's E-wide "
                         "row segment per event, YLT, offsets (north-star accounting; > 1 "
                         "because the rows are L2 hits, not HBM reads)"}
    kern = info.last_kernel.decode()
    ent = ncu_entry(kern, spec.name + ("+hoist" if args.hoist else ""))
    traffic = ent["dram_bytes_per_launch"] if ent and ent.get("n_trials") == n_loc else None
    physical = None
    if ent:
        physical = {k: ent[k] for k in ("dram_bytes_per_launch", "l2_to_l1_bytes", "l2_hit_rate",
                                        "l1_data_pipe_busy", "l1_to_l2_request_busy",
                                        "lts_throughput", "fp64_pipe", "alu_pipe",
                                        "issue_active", "warps_per_sm", "bound") if k in ent}
        physical["source"] = "profiles/scan_traffic.json (ncu --set full of this kernel " \
                             "instantiation built from these sources)"
    if args.hoist:
        # the hoisted pass: one L1/L2 read of the per-event table per (occurrence, layer)
        U = ctx.ara_layer_store_shape(0)[0]
        hb = n_ev * (4 + vb * L) + U * L * (vb * E + vb) + 8 * n_loc * L + 8 * (n_loc + 1)
        return {"bound": "hbm", "unit": "GB/s", "achieved": hb / t / 1e9, "peak": peak_hbm,
                "frac": hb / t / 1e9 / peak_hbm, "traffic": traffic, "kernel": kern,
                "kernel_ms": scan_ms, "bytes_alg_per_launch": hb, "peak_source": peak_src,
                "bytes_model": f"n*k*(4 + {vb}*L) + U*L*({vb}*E + {vb}) + 8*n*L + 8*(n+1): "
                               "hoisted-scan accounting (ids, one per-event layer loss per "
                               "occurrence and layer, the table build, YLT, offsets)",
                "physical": physical, "north_star_frac": None}
    ceil_ev, ceil_src = gather_ceiling()
    row_b = info.gather_row_bytes
    gathered = n_ev * row_b
    peak = ceil_ev * 128 / 1e9 if ceil_ev else None
    achieved = gathered / t / 1e9
    alu = None
    if args.precision == 64:
        ops = (5 * E + 9) * n_ev * L
        alu_peak = 148 * 64 * 1.965e9
        alu = {"unit": "fp64 lane-ops/s", "ops_per_trial_event": 5 * E + 9,
               "achieved": ops / t, "peak": alu_peak, "frac": ops / t / alu_peak,
               "peak_source": "148 SMs x 64 fp64 lanes/clk x 1965 MHz (nominal)"}
    return {"bound": "l2_gather", "unit": "GB/s", "achieved": achieved, "peak": peak,
            "frac": achieved / peak if peak else None, "traffic": traffic,
            "kernel": kern, "kernel_ms": scan_ms,
            "bytes_gathered_per_launch": gathered,
            "bytes_model": f"n*k*{row_b}: every trial-event gathers its {row_b}-byte row "
                           "segment(s) from the L2-resident store",
            "peak_source": f"{ceil_src} ({ceil_ev:.3e} random 128-byte row gathers/s from "
                           "L2; tools/microbench_rowpattern.cu)" if ceil_ev else None,
            "north_star_frac": ns["frac"], "north_star": ns, "alu": alu, "physical": physical}


def l2_note(info, spec) -> str:
    rows = {0: "dense event-major rows through the 8 MB catalogue map",
            1: "rows indexed by catalogue id (a (C+1)-row direct store; only the layer's "
               "events' rows are touched)",
            2: "rows indexed by catalogue id behind a 64 KB shared-memory presence bitmap "
               "(a (C+1)-row direct store; only present events' rows are touched)"}
    return (f"inputs larger than L2: the YET ({spec.n_trials} x {spec.k_max} ids) is streamed "
            f"from HBM every step; the scan reads {rows.get(info.row_addressing, '?')}; the "
            f"touched rows ({info.gather_row_bytes} B per event) are L2-resident")


def oracle_run(ds, off, ev, precision: int = 64):
    """The oracle over the whole YET on every host core: (YLT, seconds, DAT-build seconds,
    threads).  Its direct access tables are built inside the call (the paper's preprocessing,
    PAPER.md L61); that cost is measured with a 1-trial run and reported separately."""
    import oracle
    threads = max(1, len(os.sched_getaffinity(0)))
    off1 = np.ascontiguousarray(off[:2])
    t0 = time.perf_counter()
    oracle.run_analysis(ds, n_threads=threads, trial_offsets=off1 - off1[0],
                        events=ev[int(off[0]):int(off[1])], precision=precision)
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    ylt = oracle.run_analysis(ds, n_threads=threads, trial_offsets=off, events=ev,
                              precision=precision)
    return ylt, time.perf_counter() - t0, t_build, threads


def compare_parity(got, want, res, L: int, kernel: str) -> dict:
    """Every YLT entry of the last timed step against the oracle (bit-identical is the design
    target; the north star's bar is |g - o| <= 1e-9 |o| and o = 0 => g = 0), and that step's
    PML/TVaR against oracle.metrics of the oracle YLT (PML exact, TVaR within 1e-9)."""
    import oracle
    g, o = got.ravel(), want.ravel()
    nz = o != 0
    rel = np.abs(g[nz] - o[nz]) / np.abs(o[nz])
    rows = [want[l] for l in range(L)] + ([oracle.portfolio_row(want)] if L > 1 else [])
    pml_rel, tvar_rel, pml_exact = 0.0, 0.0, True
    for i, row in enumerate(rows):
        opml, otvar = oracle.metrics(row, P)
        gpml, gtvar = np.asarray(res[i][0]), np.asarray(res[i][1])
        pml_exact &= bool(np.array_equal(gpml, opml))
        pml_rel = max(pml_rel, float(np.max(np.abs(gpml - opml) / np.maximum(np.abs(opml), 1e-300))))
        tvar_rel = max(tvar_rel, float(np.max(np.abs(gtvar - otvar) / np.maximum(np.abs(otvar), 1e-300))))
    out = {"ylt_n": int(o.size), "ylt_mismatches": int(np.count_nonzero(g != o)),
           "ylt_max_rel": float(rel.max()) if rel.size else 0.0,
           "ylt_zero_flips": int(np.count_nonzero((o == 0) & (g != 0))),
           "pml_exact": pml_exact, "pml_max_rel": pml_rel, "tvar_max_rel": tvar_rel,
           "metric_rows": len(rows), "return_periods": list(RETURN_PERIODS), "tol_rel": 1e-9,
           "step": "the last timed step (steady-state kernel: " + kernel + ")",
           "oracle": "oracle/oracle.c over every trial of the workload (host threads)"}
    out["pass"] = (out["ylt_max_rel"] <= 1e-9 and out["ylt_zero_flips"] == 0 and
                   pml_rel <= 1e-9 and tvar_rel <= 1e-9)
    return out


def cpu_baseline_from(spec, ds, off, t_or, t_build, threads, per_core=True):
    """cpu_baseline from the parity oracle run (the whole workload on every host core) plus the
    per-core rate of a ~2 s one-thread slice."""
    import oracle
    n_ev = int(off[-1] - off[0])
    work = max(t_or - t_build, 1e-9)
    value = n_ev * spec.n_layers / work
    per_core_value = None
    if per_core:
        k = (spec.k_min + spec.k_max) // 2
        n1 = max(1, min(spec.n_trials, int(2.0 * value / threads / max(1, k * spec.n_layers))))
        o1, e1 = datagen.generate_yet(spec, ds.pool, 0, n1)
        t0 = time.perf_counter()
        oracle.run_analysis(ds, n_threads=1, trial_offsets=o1, events=e1)
        t1 = time.perf_counter() - t0
        per_core_value = int(o1[-1]) * spec.n_layers / max(t1 - t_build, 1e-9)
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
            "per_core_value": per_core_value,
            "sample": f"all {len(off) - 1} trials of the {spec.name} workload ({n_ev * spec.n_layers} "
                      f"trial-events); oracle/oracle.c with {threads} threads: {t_or:.1f} s, minus "
                      f"{t_build:.2f} s of direct-access-table build (preprocessing); the same run "
                      "is the parity reference"}


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    # NVML clock-event reason bits (the values nvidia-smi's clocks_event_reasons.* report)
    NVML_REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
                    0x4: "sw_power_cap"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/ara_clocks_{os.getpid()}.csv"
        self.nvml_rows = []
        self.thread = None

    def _nvml_sample(self):
        import pynvml
        sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        bits = (pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                if hasattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons")
                else pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(self.h))
        self.nvml_rows.append((float(sm), float(self.mx), bits))

    def _nvml_poll(self):
        # nvidia-smi needs ~100 ms to start, about half a timed region: NVML (the library behind
        # nvidia-smi) is also polled every 10 ms from a thread, and sampled once more when the
        # region ends (short regions)
        try:
            while not self.stop.wait(0.01):
                self._nvml_sample()
        except Exception:
            pass

    def __enter__(self):
        import threading
        self.stop = threading.Event()
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.thread = threading.Thread(target=self._nvml_poll, daemon=True)
            self.thread.start()
        except Exception:
            self.h = None
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.thread:
            self.thread.join(timeout=5)
        if self.h is not None:
            try:
                self._nvml_sample()
                import pynvml
                pynvml.nvmlShutdown()
            except Exception:
                pass
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        nv = [(sm, mx, sorted(n for b, n in self.NVML_REASONS.items() if bits & b))
              for sm, mx, bits in self.nvml_rows]
        if not self.proc and not nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0,
                    "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in (open(self.path) if self.proc else ()):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = [(sm, mx, [names[i] for i, v in enumerate(r) if v.lower() == "active"])
                for sm, mx, r in rows]
        smi_n = len(rows)
        rows += nv
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "samples": 0, "reasons": ["no samples"]}
        reasons = sorted({x for _, _, r in rows for x in r})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": rows[0][1],
                "samples": len(rows), "samples_nvidia_smi": smi_n, "samples_nvml": len(nv),
                "reasons": reasons}


def cpu_baseline_measure(spec, ds_host_elts, target_s: float = 15.0, per_core: bool = True):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload.

    The sample grows until one run takes about ``target_s``.  The oracle builds its direct access
    tables (the paper's preprocessing stage) inside every call; that cost is measured with a
    1-trial run and subtracted, as the GPU store build (A1) is outside the GPU's timed step."""
    import oracle
    threads = max(1, len(os.sched_getaffinity(0)))
    k = (spec.k_min + spec.k_max) // 2

    def run(n_tr, nt=threads):
        off, ev = datagen.generate_yet(spec, ds_host_elts.pool, 0, n_tr)
        t0 = time.perf_counter()
        oracle.run_analysis(ds_host_elts, n_threads=nt, trial_offsets=off, events=ev)
        return time.perf_counter() - t0, int(off[-1])

    t_build, _ = run(1)
    n_tr = max(threads, 64)
    while True:
        t, n_ev = run(n_tr)
        if t - t_build >= target_s / 8 or n_tr >= spec.n_trials:
            break
        n_tr = min(spec.n_trials, n_tr * 4)
    scale = target_s / max(t - t_build, 1e-3)
    if scale > 1.5 and n_tr < spec.n_trials:
        n_tr = int(min(spec.n_trials, n_tr * scale))
        t, n_ev = run(n_tr)
    work = max(t - t_build, 1e-9)
    value = n_ev * spec.n_layers / work
    # one thread on a ~2 s slice: the per-core rate (the paper's sequential C++ did
    # 2.96e6 trial-events/s on one i7-2600 core)
    per_core_value = None
    if per_core:
        n1 = max(1, min(spec.n_trials, int(2.0 * value / threads / max(1, k * spec.n_layers))))
        t1, n_ev1 = run(n1, 1)
        per_core_value = n_ev1 * spec.n_layers / max(t1 - t_build, 1e-9)
    return {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
            "per_core_value": per_core_value,
            "sample": f"first {n_tr} trials x {k} events of the {spec.name} workload "
                      f"({n_ev * spec.n_layers} trial-events, {spec.n_layers} layer(s)); "
                      f"oracle/oracle.c with {threads} threads: {t:.1f} s, minus {t_build:.2f} s "
                      f"of direct-access-table build (preprocessing)"}


def run_reference(args, spec):
    """--impl reference: the oracle (this tier's reference arm) timed on the host cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    ds = datagen.generate(spec, with_yet=False)
    # each step a bounded sample: the whole --steps K --warmup W run stays near two minutes
    per_step = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    cb = None
    vals = []
    for i in range(args.warmup + args.steps):
        cb = cpu_baseline_measure(spec, ds, target_s=min(per_step, 30.0),
                                  per_core=i == args.warmup + args.steps - 1)
        if i >= args.warmup:
            vals.append(cb["value"])
    value = statistics.median(vals)
    cb["value"] = value
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload_name(spec),
                                            "parallelism": "host threads (oracle)"},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="headline", choices=sorted(datagen.PRESETS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32],
                    help="64: the graded fp64 path; 32: the paper's float variant (F3)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="strong: the workload's n_trials split over the ranks (default; the "
                         "paper's decomposition); weak: n_trials per rank (N x n in total)")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the full-size oracle comparison of the last timed step")
    ap.add_argument("--hoist", action="store_true",
                    help="ARA_RUN_HOIST: Alg. 1 lines 4-17 once per distinct event per run, then "
                         "one table read per occurrence (SURVEY.md 7 deferred exact lever; "
                         "reported separately from the full per-occurrence scan)")
    ap.add_argument("--metrics", default="gather", choices=["gather", "sharded"],
                    help="N > 1: gather the YLT slices and compute PML/TVaR on every rank (north "
                         "star), or ara_metrics_sharded (histograms all-reduced per pass)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-offload", action="store_true",
                    help="N > 1: every rank computes PML/TVaR on the gathered YLT and the trials "
                         "split evenly (default: rank 0 alone, with a lighter trial share)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--json-out", default=None)
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    spec = datagen.PRESETS[args.config]
    if args.impl == "reference":
        return run_reference(args, spec)

    import torch
    import torch.distributed as dist

    from paper_1308_2572_b200 import ara

    rank, world, local = dist_env()
    if world != args.gpus:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}; using {world}")
    # Test hook: ARA_BENCH_SAME_DEVICE=1 puts every rank on cuda:0 over gloo (NCCL refuses two
    # ranks on one GPU), so the multi-rank path can be exercised on a 1-GPU box.
    same_dev = os.environ.get("ARA_BENCH_SAME_DEVICE") == "1"
    if same_dev:
        local = 0
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    if world > 1:
        if same_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    # ---- inputs: ELTs/layers are identical on every rank (seeded); each rank generates only
    # its own trial slice of the YET (counter-based substreams), so the YET is never sent.
    ds = datagen.generate(spec, with_yet=False)
    from paper_1308_2572_b200 import dist as adist
    if world > 1:  # setup collective: rank 0's ELTs and terms reach every rank (NVLink)
        adist.broadcast_inputs(ds, src=0)
    n_total = spec.n_trials * world if args.scaling == "weak" else spec.n_trials
    L = ds.n_layers
    # YLT rows 0..L-1 and, for L > 1, the portfolio-scope row L
    L1 = L + 1 if L > 1 else L
    parts = adist.partition_trials(n_total, world)  # balanced contiguous ranges

    def load_slice(parts):
        """This rank's YET slice (host, pinned) and its device copies and YLT buffers."""
        t0, t1 = parts[rank]
        n_loc = t1 - t0
        h_off_np = datagen.trial_offsets(spec, t0, n_loc)
        n_ev = int(h_off_np[-1])
        h_ids = torch.empty(n_ev, dtype=torch.int32, pin_memory=True)
        datagen.generate_yet(spec, ds.pool, t0, n_loc, out=h_ids.numpy().view(np.uint32))
        h_off = torch.from_numpy(h_off_np.view(np.int64)).pin_memory()
        d_ylt_buf = torch.empty((L1, n_loc), dtype=torch.float64, device=dev)
        return (n_loc, h_off_np, n_ev, h_ids, h_off, h_off.to(dev).view(torch.uint64),
                h_ids.to(dev).view(torch.uint32), d_ylt_buf, d_ylt_buf[:L],
                d_ylt_buf[L] if L > 1 else None)

    (n_loc, h_off_np, n_ev, h_ids, h_off, d_off, d_ids, d_ylt_buf, d_ylt_loc,
     d_port_loc) = load_slice(parts)
    d_full_buf = torch.empty((L1, n_total), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    ctx = ara.Context(local, stream)
    ctx.ara_set_precision(args.precision)
    ctx.ara_load_elts(ds.catalogue_size, ds.rec_offsets, ds.rec_event_ids, ds.rec_losses, ds.fin)
    t_store = time.perf_counter()
    ctx.ara_set_layers(ds.layer_terms, ds.elt_offsets, ds.elt_index)
    t_store = time.perf_counter() - t_store
    torch.cuda.synchronize()
    if rank == 0:
        log(f"[bench] {workload_name(spec)}; ranks {world}; local trials {n_loc}; "
            f"store {ctx.ara_get_info().store_bytes / 1e6:.1f} MB built in {t_store * 1e3:.1f} ms")

    def gather():
        if world == 1:
            return d_ylt_buf
        adist.gather_ylt(d_ylt_loc, n_total, out=d_full_buf[:L], parts=parts)
        return d_full_buf

    def post_metrics(rows):
        """A9 on the gathered YLT rows (+ the portfolio row): one batched call (synchronous)."""
        if L > 1:
            ctx.ara_portfolio_ylt(rows[:L], rows[L])
        pml, tvar = ctx.ara_metrics_rows(rows[:L1], P)
        return [(pml[i], tvar[i]) for i in range(L1)]

    scan_ev = []
    run_flags = ara.ARA_RUN_HOIST if args.hoist else 0
    # Strong/weak scaling with the gathered YLT: rank 0 alone computes PML/TVaR (every rank holds
    # the same gathered rows, so one evaluation suffices), and it scans correspondingly fewer
    # trials so that no rank waits on the others (dist.partition_rank0_offload).  The metrics'
    # cost in scanned trials, mu, is measured here on the balanced split: one scan per rank and
    # one metrics call on rank 0, timed with CUDA events; the slices are then regenerated.
    offload = world > 1 and args.metrics == "gather" and not args.no_offload
    mu = 0.0
    if offload:
        for _ in range(2):
            ctx.ara_run(d_off, d_ids, d_ylt_loc, flags=run_flags)
        rows = gather()
        post_metrics(rows)
        torch.cuda.synchronize()
        ta = torch.cuda.Event(enable_timing=True); tb = torch.cuda.Event(enable_timing=True)
        ta.record(stream)
        for _ in range(3):
            ctx.ara_run(d_off, d_ids, d_ylt_loc, flags=run_flags)
        tb.record(stream)
        torch.cuda.synchronize()
        t_trial = ta.elapsed_time(tb) / 3 / max(n_loc, 1)
        rows = gather()
        t_met = 0.0
        if rank == 0:
            torch.cuda.synchronize()
            ta.record(stream)
            for _ in range(3):
                post_metrics(rows)
            tb.record(stream)
            torch.cuda.synchronize()
            t_met = ta.elapsed_time(tb) / 3
        t_trial, t_met = adist.max_over_ranks([t_trial, t_met])
        mu = t_met / t_trial if t_trial > 0 else 0.0
        parts = adist.partition_rank0_offload(n_total, world, mu)
        (n_loc, h_off_np, n_ev, h_ids, h_off, d_off, d_ids, d_ylt_buf, d_ylt_loc,
         d_port_loc) = load_slice(parts)
        if rank == 0:
            log(f"[bench] metrics on rank 0 = {t_met:.3f} ms = {mu:.0f} trials of scanning; "
                f"trials per rank {[b - a for a, b in parts]}")

    def step(timed: bool):
        if timed:
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
        ctx.ara_run(d_off, d_ids, d_ylt_loc, flags=run_flags)  # A2-A8: one fused scan launch
        if timed:
            b.record(stream)
            scan_ev.append((a, b))
        if world > 1 and args.metrics == "sharded":
            res = [adist.sharded_metrics(ctx, d_ylt_loc[l], n_total, P) for l in range(L)]
            if L > 1:  # portfolio scope: per-trial sum over layers
                ctx.ara_portfolio_ylt(d_ylt_loc, d_port_loc)
                res.append(adist.sharded_metrics(ctx, d_port_loc, n_total, P))
            return res
        rows = gather()
        if offload and rank != 0:
            return None
        return post_metrics(rows)  # A9 (+ portfolio scope)

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    ctx.ara_synchronize()

    launches0 = ctx.kernel_launches
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            res = step(True)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ctx.ara_synchronize()
    launches = ctx.kernel_launches - launches0
    # the last timed step's YLT (gathered over the ranks), for the parity check below
    if world > 1 and args.metrics == "sharded" and not args.no_parity:  # not gathered in steps
        adist.gather_ylt(d_ylt_loc, n_total, out=d_full_buf[:L], parts=parts)
    last_ylt = (d_full_buf if world > 1 else d_ylt_buf)[:L].cpu().numpy() if rank == 0 else None
    ms = e0.elapsed_time(e1) / args.steps
    scan_ms = statistics.mean(a.elapsed_time(b) for a, b in scan_ev)
    if world > 1:
        ms, scan_ms = adist.max_over_ranks([ms, scan_ms])

    # every rank's events (weak scaling: N slices of the workload; strong: one split over ranks)
    n_ev_all = n_ev
    if world > 1:
        n_ev_all = int(adist.sum_over_ranks([float(n_ev)])[0])
    trial_events = n_ev_all * spec.n_layers
    value = trial_events / (ms * 1e-3)
    info = ctx.ara_get_info()
    last_kernel = info.last_kernel.decode()
    E = spec.elts_per_layer
    rf = roofline(args, spec, ctx, info, n_ev, n_loc, scan_ms)

    # ---- end to end through the host-buffer C-ABI call
    e2e = None
    if not args.no_e2e:
        # every host buffer pinned (the YET, its offsets and the YLT): pageable buffers would be
        # staged through a bounce buffer by the driver
        h_ylt_t = torch.empty((L, n_loc), dtype=torch.float64, pin_memory=True)
        h_ylt = h_ylt_t.numpy()
        ids_np = h_ids.numpy().view(np.uint32)
        off_np = h_off.numpy().view(np.uint64)
        for _ in range(2):
            ctx.ara_run_host(off_np, ids_np, h_ylt, flags=run_flags)
        ts = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            tt = time.perf_counter()
            ctx.ara_run_host(off_np, ids_np, h_ylt, flags=run_flags)  # H2D YET, scan, D2H YLT
            d_ylt_loc.copy_(h_ylt_t, non_blocking=False)
            if world > 1 and args.metrics == "sharded":
                for l in range(L):
                    adist.sharded_metrics(ctx, d_ylt_loc[l], n_total, P)
                if L > 1:
                    ctx.ara_portfolio_ylt(d_ylt_loc, d_port_loc)
                    adist.sharded_metrics(ctx, d_port_loc, n_total, P)
            else:
                rows = gather()
                if not (offload and rank != 0):
                    post_metrics(rows)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - tt)
        t_e2e = statistics.median(ts)
        if world > 1:
            t_e2e = adist.max_over_ranks([t_e2e])[0]
        h2d = (n_loc + 1) * 8 + n_ev * 4 + L * n_loc * 8
        d2h = L * n_loc * 8 + L * len(P) * 16
        e2e = {"value": trial_events / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": t_e2e * 1e3,
               "note": "ara_run_host (pinned host YET + offsets -> device in 64 MiB chunks overlapped with "
                       "the scan, YLT back to host) + YLT upload + ara_metrics; wall clock, "
                       "median of steps, max over ranks"}

    # ---- parity of the last timed step (its YLT is still in the buffers) against the oracle run
    # over every trial of the workload; the same run is the CPU baseline (rank 0)
    parity, cpu = None, None
    if rank == 0 and not (args.no_parity and (args.no_cpu_baseline or world > 1)):
        got = last_ylt
        if world > 1:  # rank 0 regenerates the whole YET (counter-based: identical trials)
            off_all, ev_all = datagen.generate_yet(spec, ds.pool, 0, n_total)
        else:
            off_all, ev_all = h_off_np, h_ids.numpy().view(np.uint32)
        want, t_or, t_build, threads = oracle_run(ds, off_all, ev_all, args.precision)
        if not args.no_parity:
            parity = compare_parity(got, want, res, L, last_kernel)
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_from(spec, ds, off_all, t_or, t_build, threads,
                                    per_core=True)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64" if args.precision == 64 else "f32",
            "data": "synthetic (datagen SplitMix64, seed 1308; truncated-Pareto ELT losses)",
            "config": {"variant": ("hoisted (ARA_RUN_HOIST: per-event layer losses once per "
                                   "distinct event per run; SURVEY.md 7 deferred exact lever)"
                                   if args.hoist else "full per-occurrence scan (north star)"),
                       "workload": workload_name(spec) + (
                           f" per GPU ({n_total} trials in total)"
                           if world > 1 and args.scaling == "weak" else ""), "layers": L, "elts_per_layer": E,
                       "trials": n_total, "trials_per_gpu": n_loc,
                       "trials_by_rank": [b - a for a, b in parts] if world > 1 else None,
                       "metrics_on": ("rank 0 (rank 0 scans fewer trials: the metrics cost "
                                      f"{mu:.0f} trials of scanning, measured)" if offload
                                      else "every rank" if world > 1 else "the GPU"),
                       "events_per_trial": spec.k_min,
                       "parallelism": f"trial-sharded x{world}, {args.scaling} scaling "
                                      + ("(PML/TVaR by sharded radix select, histograms "
                                         "all-reduced per pass)" if args.metrics == "sharded"
                                         else f"({dist.get_backend().upper()} all-gather of "
                                              "the YLT for PML/TVaR)")
                       if world > 1 else "1 GPU",
                       "l2": l2_note(info, spec),
                       "return_periods": list(RETURN_PERIODS)},
            "roofline": rf,
            "parity": parity,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "pml": res[0][0].tolist(), "tvar": res[0][1].tolist(),
            "pml_portfolio": res[L][0].tolist() if L > 1 else None,
            "tvar_portfolio": res[L][1].tolist() if L > 1 else None,
        }
        s = json.dumps(line)
        print(s, flush=True)
        if args.json_out:
            with open(args.json_out, "w") as f:
                f.write(s + "\n")
    if world > 1:
        dist.barrier()  # rank 0's oracle run may outlast the others' teardown
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
