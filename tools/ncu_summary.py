"""Key counters of an ncu capture (exported with --page raw --csv) as markdown.

    ncu -i prof.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_summary.py raw.csv [label] >> profiles/r01_ncu.md
"""

from __future__ import annotations

import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (warp-inst/clk/SM)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "FMA-heavy pipe cycles %"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps / scheduler"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe cycles %"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall: math pipe throttle"),
    ("smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio", "stall: dispatch"),
    ("smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio", "stall: not selected"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait (fixed latency)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def main(path: str, label: str = "") -> None:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "gpu__time_duration.sum" in r)
    hdr, units = rows[hi], rows[hi + 1]
    for vals in rows[hi + 2:]:
        if len(vals) < len(hdr):
            continue
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "kernel"
        print(f"\n#### {label} `{name}`\n")
        print("| counter | value |")
        print("|---|---|")
        for k, desc in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"| {desc} (`{k}`) | {vals[i]} {units[i]} |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
