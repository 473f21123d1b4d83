"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes) per kernel name."""
import collections
import csv
import sys


def main(path, top=20, steps=1):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[1:]:
        name = r[ki].split("(")[0][:60]
        agg[name][r[mi]] += float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            cnt[name] += 1
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"])[:top]:
        t = a["gpu__time_duration.sum"]
        print(f"{n:60s} n={cnt[n]:5d} {t / 1e6 / steps:9.2f} ms/step {100 * t / tot:5.1f}% "
              f"rd {a['dram__bytes_read.sum'] / 1e9 / steps:8.2f} GB wr {a['dram__bytes_write.sum'] / 1e9 / steps:7.2f} GB")
    print(f"total {tot / 1e6 / steps:.2f} ms/step")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20, float(sys.argv[3]) if len(sys.argv) > 3 else 1)
