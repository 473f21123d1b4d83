#!/usr/bin/env python3
"""Throughput of the device text loader (cs_db_load_text) on a seeded CSV of cfg2's shape.

    python tools/bench_ingest.py [--m 1000000] [--n 100] [--steps 5] [--warmup 3]

Prints one JSON line: ``value`` = text GB/s with the text already in HBM (device input; the
loader's own scans, host syncs and allocations are inside the timed region), ``e2e`` = the
same from a host buffer (H2D copy inside), ``roofline`` against the measured HBM peak with
algorithmic bytes = text bytes read + column bytes written, ``cpu_baseline`` = this package's
host restatement of the reference's load_csv (pure Python, as the reference) on a bounded
sample of the rows.
"""

from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def make_text(n, m, seed=5):
    rng = np.random.default_rng(seed)
    ar = rng.integers(2, 6, size=n)
    x = (rng.random((m, n)) * ar).astype(np.uint8)
    # fast printing: every state is one digit
    body = np.full((m, 2 * n), ord(","), dtype=np.uint8)
    body[:, 0::2] = x + ord("0")
    body[:, -1] = ord("\n")
    return x.T.copy(), body.tobytes()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1_000_000)
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cpu-rows", type=int, default=100_000)
    args = ap.parse_args()

    import torch

    import paper_1804_04640_b200 as cs
    from paper_1804_04640_b200.engine import GpuDatabase

    x, text = make_text(args.n, args.m)
    ctx = cs.shared_context(0)
    host = torch.from_numpy(np.frombuffer(text, dtype=np.uint8).copy()).pin_memory()  # e2e source
    pageable = np.frombuffer(text, dtype=np.uint8)
    dev = host.cuda()
    l0 = ctx.launches
    gdb = GpuDatabase.from_text(ctx, dev)
    launches = ctx.launches - l0
    ok = all(np.array_equal(gdb.download(i), x[i]) for i in range(0, args.n, max(1, args.n // 10)))
    gdb.close()
    assert ok, "device loader output differs from the printed matrix"

    def timed(src):
        for _ in range(args.warmup):
            GpuDatabase.from_text(ctx, src).close()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            g = GpuDatabase.from_text(ctx, src)
            ctx.sync()
            ts.append(time.perf_counter() - t0)
            g.close()
        return float(np.median(ts))

    t_dev = timed(dev)
    t_host = timed(host)
    t_pageable = timed(pageable)
    nbytes = len(text)
    algo = nbytes + args.n * args.m
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0

    # CPU: the reference's load_csv as restated on the host (pure Python tokeniser)
    rows = min(args.cpu_rows, args.m)
    with tempfile.TemporaryDirectory() as td:
        p = Path(td) / "s.csv"
        p.write_bytes(text[: rows * 2 * args.n])
        t0 = time.perf_counter()
        cs.load_csv(p)
        t_cpu = time.perf_counter() - t0
    cpu_gbs = rows * 2 * args.n / t_cpu / 1e9

    print(json.dumps({
        "metric": "csv ingest text GB/s", "value": nbytes / t_dev / 1e9, "unit": "GB/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev * 1e3, "higher_is_better": True,
        "dtype": "u8", "data": "synthetic (seeded, one-digit states, ',' separated)",
        "config": {"workload": "csv ingest", "n": args.n, "m": args.m, "text_bytes": nbytes},
        "roofline": {"bound": "hbm", "achieved": algo / t_dev / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": algo / t_dev / 1e9 / peak, "traffic": None,
                     "note": "whole loader call incl. host syncs and scratch allocation; algorithmic bytes = text + columns"},
        "e2e": {"value": nbytes / t_host / 1e9, "unit": "GB/s", "h2d_bytes_per_step": nbytes,
                "d2h_bytes_per_step": 4 * args.n + 64, "ms_per_step": t_host * 1e3,
                "pageable_gbs": nbytes / t_pageable / 1e9},
        "gpu_launches": launches,
        "cpu_baseline": {"value": cpu_gbs, "unit": "GB/s", "cores": 1, "kind": "port",
                         "sample": f"first {rows} rows through the host load_csv restatement in {t_cpu:.1f} s"},
    }))


if __name__ == "__main__":
    main()
