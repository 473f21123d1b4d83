#!/usr/bin/env python3
"""Host-side plan build time vs CS_PLAN_THREADS on the cfg3 subset batch (74,518 queries)."""
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

if len(sys.argv) > 1:
    import numpy as np

    import paper_1804_04640_b200 as cs
    from paper_1804_04640_b200 import workloads as W
    from paper_1804_04640_b200.engine import FamilyScorer, QueryPlan

    w = W.cfg3()
    ctx = cs.shared_context(0)
    gdb = w.build_device(ctx)
    fams = [(q[0], tuple(q[1:])) for q in w.queries]
    fs = FamilyScorer(gdb, fams)
    from paper_1804_04640_b200.engine import encode_queries

    off, flat = encode_queries(fs.subsets)
    out = np.zeros(len(fs.subsets))
    for _ in range(2):
        gdb.query_batch(off, flat, cs._native.CS_NLOGN, loglik=out)
    t0 = time.perf_counter()
    for _ in range(5):
        gdb.query_batch(off, flat, cs._native.CS_NLOGN, loglik=out)
    print(f"threads={os.environ.get('CS_PLAN_THREADS')} one-shot {(time.perf_counter() - t0) / 5 * 1e3:.2f} ms "
          f"nq={len(fs.subsets)} cpus={os.cpu_count()} affinity={len(os.sched_getaffinity(0))}")
else:
    for t in ("1", "2", "4", "8"):
        env = dict(os.environ, CS_PLAN_THREADS=t, CS_TRACE="1")
        r = subprocess.run([sys.executable, __file__, "x"], env=env, capture_output=True, text=True)
        print(r.stdout.strip())
        print("\n".join(r.stderr.strip().splitlines()[-4:]))
