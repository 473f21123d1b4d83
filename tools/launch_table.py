#!/usr/bin/env python3
"""Per-kernel totals of an ncu --metrics launch list (time, DRAM bytes, achieved DRAM GB/s).

    python tools/launch_table.py launches.csv [--skip-until REGEX]
"""
import collections
import csv
import io
import sys


def main(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        if unit == "ns":
            v *= 1e-3
        elif unit == "ms":
            v *= 1e3
        elif unit == "us":
            pass
        elif unit in ("Kbyte", "KB"):
            v *= 1e3
        elif unit in ("Mbyte", "MB"):
            v *= 1e6
        elif unit in ("Gbyte", "GB"):
            v *= 1e9
        per[r["ID"]][r["Metric Name"]] = v
        names[r["ID"]] = r["Kernel Name"].split("(")[0]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, mets in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += mets.get("gpu__time_duration.sum", 0.0)
        a[2] += mets.get("dram__bytes_read.sum", 0.0)
        a[3] += mets.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values()) or 1.0
    print("| kernel | launches | total us | share | DRAM read MB | DRAM write MB | DRAM GB/s |")
    print("|---|---|---|---|---|---|---|")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = (a[2] + a[3]) / (a[1] * 1e-6) / 1e9 if a[1] else 0.0
        print(f"| `{k}` | {a[0]} | {a[1]:.0f} | {100 * a[1] / tot:.1f}% | {a[2] / 1e6:.1f} | {a[3] / 1e6:.1f} | {gbs:.0f} |")
    print(f"\ntotal {tot:.0f} us over {sum(a[0] for a in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
