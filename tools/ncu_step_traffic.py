#!/usr/bin/env python3
"""Timed-step view of an ncu launch list from tools/ncu_traffic.sh (bench --steps 1 --warmup 3).

The bench's device-timed step repeats the same launch sequence; the smallest period L with
names[0:L] == names[L:2L] == names[2L:3L] == names[3L:4L] is one step, and launches [3L, 4L) are
the timed one (the e2e leg that follows plans differently and is ignored).  Prints per-kernel
totals of that step and a JSON line: {"config", "launches", "time_ms", "dram_bytes", "dram_gbs"}.

    python tools/ncu_step_traffic.py gpurun_out/s3/cfg2_launches.csv cfg2
"""
import collections
import csv
import io
import json
import sys

SCALE = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
         "byte": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}


def load(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    per = collections.OrderedDict()
    for r in rows:
        i = int(r["ID"])
        d = per.setdefault(i, {"name": r["Kernel Name"].split("(")[0].split("<")[0].strip(),
                               "full": r["Kernel Name"] + r["Grid Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1.0)
    return [per[i] for i in sorted(per)]


def main(path, config):
    ls = load(path)
    names = [x["full"] for x in ls]
    L = next(L for L in range(1, len(names) // 4 + 1)
             if names[0:L] == names[L:2 * L] == names[2 * L:3 * L] == names[3 * L:4 * L])
    step = ls[3 * L:4 * L]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for x in step:
        a = agg[x["name"]]
        a[0] += 1
        a[1] += x.get("gpu__time_duration.sum", 0.0)
        a[2] += x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
    t = sum(a[1] for a in agg.values())
    b = sum(a[2] for a in agg.values())
    for k, (n, ms, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:28s} {n:5d} launches {ms:9.3f} ms ({100 * ms / t:5.1f}%)  dram {by / 1e9:8.3f} GB  "
              f"{by / (ms * 1e-3) / 1e9 if ms else 0:8.1f} GB/s")
    print(json.dumps({"config": config, "launches": len(step), "time_ms": t, "dram_bytes": b,
                      "dram_gbs": b / (t * 1e-3) / 1e9}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
