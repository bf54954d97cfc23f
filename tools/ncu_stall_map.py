#!/usr/bin/env python3
"""Source-level (SASS) warp-stall map of one kernel from an `ncu --set full --import-source on`
report: stall reasons over the launch, executed warp instructions by opcode (per unit of work when
--units is given), and the hottest instructions.  Reads `ncu -i REPORT --page source --csv
--print-source sass` (the ncu CLI runs without a GPU).

    python tools/ncu_stall_map.py REPORT.ncu-rep [--units 1e9 --unit-name trial-event] [--top 15]
"""
import argparse
import collections
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--units", type=float, default=0.0, help="units of work per launch")
    ap.add_argument("--unit-name", default="unit")
    ap.add_argument("--top", type=int, default=15)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    kernel = rows[0][1] if rows and rows[0] and rows[0][0] == "Kernel Name" else "?"
    h = rows[1]
    data = [r for r in rows[2:] if len(r) == len(h)]
    col = {name: i for i, name in enumerate(h)}

    def num(r, name):
        v = r[col[name]].replace(",", "") if name in col else ""
        try:
            return float(v)
        except ValueError:
            return 0.0

    stalls = [n for n in h if n.startswith("stall_") and "(Not Issued)" not in n]
    tot = collections.Counter()
    for r in data:
        for n in stalls:
            tot[n] += num(r, n)
    all_samples = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
    print(f"# {kernel}")
    print(f"total samples {all_samples:.0f}")
    for n, v in tot.most_common():
        print(f"{n:30s} {v:10.0f} {v / max(all_samples, 1):.3f}")
    ops = collections.Counter()
    op_st = collections.Counter()
    for r in data:
        src = r[col["Source"]].strip()
        tok = src.split()
        if not tok:
            continue
        op = tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]
        op = op.split(".")[0]
        ops[op] += num(r, "Instructions Executed")
        op_st[op] += num(r, "Warp Stall Sampling (All Samples)")
    n_inst = sum(ops.values())
    print()
    per = f" (per {args.unit_name}: divide by {args.units:.3g})" if args.units else ""
    print(f"executed warp instructions by opcode{per}, share, stall samples")
    for op, v in ops.most_common(30):
        extra = f" per-{args.unit_name} {v / args.units:.4f}" if args.units else ""
        print(f"{op:12s} {v:14.0f} {v / max(n_inst, 1):.3f}  stall-samples {op_st[op]:.0f}{extra}")
    print()
    print("top stalled instructions (all samples / long-scoreboard / wait):")
    data.sort(key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))
    for r in data[:args.top]:
        print(f"  {r[col['Address']]}  {num(r, 'Warp Stall Sampling (All Samples)'):8.0f} "
              f"long={num(r, 'stall_long_sb'):8.0f} wait={num(r, 'stall_wait'):8.0f}  "
              f"{r[col['Source']].strip()}")


if __name__ == "__main__":
    main()
