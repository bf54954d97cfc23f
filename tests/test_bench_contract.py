"""bench.py contract on CPU: the reference arm (the oracle) prints one JSON line with the keys
the driver reads; the multi-rank partition helpers agree with dist.py."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "tiny", "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "trial-events/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_warmup_floor():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "tiny", "--steps", "1", "--warmup", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode != 0


def test_partition_matches_dist():
    sys.path.insert(0, ROOT)
    import bench
    from paper_1308_2572_b200.dist import partition_trials
    for n, R in ((1_000_000, 8), (10, 4), (7, 3)):
        assert [bench.partition(n, r, R) for r in range(R)] == partition_trials(n, R)


def test_clock_summary_reasons():
    """The clocks line merges nvidia-smi and NVML samples; throttle reasons are named from
    either source (a run that saw hw/thermal slowdowns must say so)."""
    sys.path.insert(0, ROOT)
    import bench
    cs = bench.ClockSampler(0)
    cs.nvml_rows = [(1965.0, 1965.0, 0), (1900.0, 1965.0, 0x4), (1965.0, 1965.0, 0x8 | 0x40)]
    s = cs.summary()
    assert s["samples"] == 3 and s["samples_nvml"] == 3 and s["samples_nvidia_smi"] == 0
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["hw_slowdown", "hw_thermal_slowdown", "sw_power_cap"]
    empty = bench.ClockSampler(0).summary()
    assert empty["sm_mhz"] is None and empty["reasons"]


@pytest.mark.gpu
def test_bench_json_line_on_gpu():
    """bench.py on the GPU (medium config, short run) prints one JSON line with every key the
    driver reads, a positive value, the roofline / e2e / clocks objects and kernel launches."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "medium",
                          "--steps", "3", "--warmup", "3", "--e2e-steps", "2"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "gpu_launches", "clocks", "e2e", "cpu_baseline"):
        assert k in d, k
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["dtype"] == "f64"
    r = d["roofline"]
    assert r["bound"] == "l2_gather" and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9 and 0 < r["frac"] <= 1.05
    assert r["north_star"]["bound"] == "hbm" and r["north_star_frac"] > 0
    assert r["kernel"].startswith(("pair_scan_kernel<", "scan_kernel<"))
    p = d["parity"]  # every YLT entry of the last timed step against the oracle
    assert p["pass"] and p["ylt_mismatches"] == 0 and p["ylt_n"] == 100_000 and p["pml_exact"]
    assert d["gpu_launches"] >= 3 * 3  # probe / length check or sort, scan, metrics per step
    assert d["e2e"]["h2d_bytes_per_step"] > 4 * 10**8 and d["e2e"]["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "sm_mhz" in d["clocks"]
