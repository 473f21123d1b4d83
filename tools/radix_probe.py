"""Probe the partition class (k_radix_part + k_radix_count) on cfg5-shaped big tables.

    python tools/radix_probe.py [--m 100000000] [--nq 64] [--reps 3]

Builds a cfg5-shaped database (arity U{2..8}) with n=40 variables on the device, plans only
queries whose tables exceed SMEM capacity, and prints the device time of the histogram phase
(library CUDA events) with the algorithmic bytes (k*m per query, uint8 convention) per second.
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200 import workloads  # noqa: E402
from paper_1804_04640_b200.engine import QueryPlan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=100_000_000)
    ap.add_argument("--nq", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--kmin", type=int, default=2)
    a = ap.parse_args()
    ctx = cs.shared_context(0)
    w = workloads.cfg5(seed=5, nq=20000, m=a.m, n=40)
    qs = [q for q in w.queries if len(q) >= a.kmin and np.prod([int(w.arities[v]) for v in q]) > 56_320][:a.nq]
    t0 = time.time()
    gdb = w.build_device(ctx)
    ctx.sync()
    print(f"db built in {time.time() - t0:.1f} s; {len(qs)} queries, mean k {np.mean([len(q) for q in qs]):.2f}, "
          f"median C {np.median([np.prod([int(w.arities[v]) for v in q]) for q in qs]):.0f}", flush=True)
    plan = QueryPlan(gdb, qs)
    ll = np.zeros(plan.nq)
    byts = sum(len(q) for q in qs) * a.m
    for r in range(a.reps + 1):
        plan.execute(loglik=ll)
        ms = ctx.last_kernel_ms()
        if r:
            print(f"rep {r}: {ms:.2f} ms  {byts / ms / 1e6:.0f} GB/s logical  {ms * 1e3 / len(qs):.0f} us/query", flush=True)


if __name__ == "__main__":
    main()
