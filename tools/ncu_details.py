#!/usr/bin/env python3
"""Print the key sections of an `ncu --page details --csv` export (speed of light, memory,
occupancy, scheduler, warp state) and selected raw metrics of a `--page raw --csv` export."""
import csv
import io
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy",
            "Scheduler Statistics", "Warp State Statistics", "Compute Workload Analysis")
RAW = ["smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
       "smsp__inst_executed_pipe_alu.sum", "smsp__inst_executed_op_shared_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
       "dram__bytes_read.sum", "lts__t_bytes.sum", "gpu__time_duration.sum"]


def details(path):
    rows = list(csv.reader(io.StringIO(open(path).read())))
    h = rows[0]
    ki, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    for r in rows[1:]:
        if len(r) > vi and r[ki] in SECTIONS and r[mi]:
            print(f"  {r[ki][:18]:18s} {r[mi]}: {r[vi]} {r[ui]}")


def raw(path):
    rows = list(csv.reader(io.StringIO(open(path).read())))
    h = rows[0]
    for w in RAW:
        if w in h:
            i = h.index(w)
            print(f"  {w}: {rows[2][i] if len(rows) > 2 else ''} {rows[1][i]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        (raw if "full_" in p or "raw" in p else details)(p)
