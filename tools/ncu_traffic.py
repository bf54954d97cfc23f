#!/usr/bin/env python3
"""Update profiles/scan_traffic.json (read by bench.py as roofline.traffic / physical) from one
`ncu --set full` capture of a scan or portfolio launch.

    python tools/ncu_traffic.py CONFIG REPORT.ncu-rep N_TRIALS "bound text" [--source TEXT]

Reads the report's raw page (ncu -i ... --page raw --csv) and stores DRAM bytes per launch
(dram__bytes_read.sum + dram__bytes_write.sum), L1 data-pipe / L1->L2 request / L2 / fp64 / ALU /
issue utilisation and the duration under ncu, keyed "<kernel instantiation>|<source hash>|
<config>" (paper_1308_2572_b200.build.source_sha16: the sources that determine libara.so's
code; nvcc output itself is not byte-reproducible): bench.py reports an entry only for the same
kernel built from the same sources, so a changed kernel never shows stale counters.  Run it on
a report of the library built from the committed sources.
"""
import csv
import io
import re
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "scan_traffic.json")

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1, "msecond": 1, "nsecond": 1e-6}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def num(d, key):
    val, unit = d[key]
    return float(val.replace(",", "")) * UNIT.get(unit, 1)


def pct(d, key):
    return float(d[key][0].replace(",", "")) / 100.0


def main():
    cfg, report, n_trials, bound = sys.argv[1:5]
    src = sys.argv[sys.argv.index("--source") + 1] if "--source" in sys.argv else report
    sys.path.insert(0, ROOT)
    from paper_1308_2572_b200.build import source_sha16
    sha = source_sha16()  # nvcc output is not byte-reproducible: key by the sources
    d = raw(report)
    m = re.search(r"(\w+<[^()]*>)\(", d["Kernel Name"][0])
    kern = m.group(1) if m else d["Kernel Name"][0]
    entry = {
        "kernel": kern,
        "src_sha16": sha,
        "n_trials": int(n_trials),
        "dram_bytes_per_launch": num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum"),
        "l2_to_l1_bytes": num(d, "l1tex__m_xbar2l1tex_read_bytes.sum"),
        "l2_hit_rate": pct(d, "lts__t_sector_hit_rate.pct"),
        "l1_data_pipe_busy": pct(d, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "l1_to_l2_request_busy": pct(d, "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "lts_throughput": pct(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_per_sm": num(d, "sm__warps_active.avg.per_cycle_active"),
        "fp64_pipe": pct(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "alu_pipe": pct(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active": pct(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warp_instructions": num(d, "smsp__inst_executed.sum"),
        "kernel_ms_under_ncu": num(d, "gpu__time_duration.sum"),
        "bound": bound,
    }
    j = json.load(open(OUT)) if os.path.exists(OUT) else {}
    j = {k: v for k, v in j.items() if "|" in k or k == "source"}  # round-1 keys were stale
    j[f"{kern}|{sha}|{cfg}"] = entry
    j["source"] = src
    with open(OUT, "w") as f:
        json.dump(j, f, indent=1)
        f.write("\n")
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main()
