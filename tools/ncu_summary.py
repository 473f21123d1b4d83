#!/usr/bin/env python3
"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/ncu_summary.py launches <launches.csv>           -> per-kernel share table
    python tools/ncu_summary.py full <prof.ncu-rep> [algo_bytes]  -> key metrics of one kernel
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "smsp__inst_executed_op_shared_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
]


def launches(path: str) -> str:
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.defaultdict(list)
    for r in rows:
        if r.get("Metric Name") == "gpu__time_duration.sum":
            agg[r["Kernel Name"].split("(")[0]].append(float(r["Metric Value"]))
    unit = rows[0].get("Metric Unit", "") if rows else ""
    total = sum(sum(v) for v in agg.values()) or 1.0
    out = [f"| kernel | launches | mean ({unit}) | total share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v):.1f} | {100 * sum(v) / total:.1f}% |")
    return "\n".join(out)


def full(path: str, algo_bytes: float | None = None) -> dict:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    if algo_bytes:
        for d in res:
            try:
                rd = float(d["dram__bytes_read.sum"].split()[0].replace(",", ""))
                unit = d["dram__bytes_read.sum"].split()[1]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
                d["algorithmic_bytes"] = algo_bytes
                d["dram_read_over_algorithmic"] = rd * scale / algo_bytes
            except Exception:
                pass
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(json.dumps(full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None), indent=1))
