#!/usr/bin/env python3
"""Side-by-side key metrics of `ncu --page raw --csv` exports (one kernel launch each).

    python tools/ncu_compare.py a_raw.csv b_raw.csv ...
"""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("l1tex__data_pipe_lsu_wavefronts.sum", "L1 data wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "  of which shared/shfl"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data pipe %"),
    ("l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_elapsed", "L1 writeback %"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->L1 bytes"),
    ("lts__t_sectors_srcunit_tex_lookup_hit.sum", "L2 hit sectors"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long sb"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg throttle"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short sb"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math throttle"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio throttle"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall not selected"),
    ("smsp__average_warps_issue_stalled_selected_per_issue_active.ratio", "selected"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall dispatch"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio", "stall branch"),
    ("smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio", "stall no inst"),
    ("smsp__average_warps_issue_stalled_drain_per_issue_active.ratio", "stall drain"),
    ("smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio", "stall imc miss"),
    ("smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio", "stall tex throttle"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "occ limit regs"),
]


def load(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr, units, vals = rows[i], rows[i + 1], rows[i + 2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def main():
    runs = [load(p) for p in sys.argv[1:]]
    w = max(len(n) for _, n in KEYS)
    for key, name in KEYS:
        cells = []
        for r in runs:
            v, u = r.get(key, ("-", ""))
            cells.append(f"{v} {u}".strip())
        print(f"{name:<{w}}  " + "  |  ".join(f"{c:>22}" for c in cells))


if __name__ == "__main__":
    main()
