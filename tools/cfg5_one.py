"""One cfg5 (m = 1e8) plan of the stream's first n queries with k variables and lo < cells <= hi,
executed twice (for ncu captures of a single class / variant).

    python tools/cfg5_one.py k lo hi [n] [flags]      flags: 1 tables (default), 0 score only
"""
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200 import workloads  # noqa: E402
from paper_1804_04640_b200.engine import QueryPlan  # noqa: E402

k, lo, hi = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
n = int(sys.argv[4]) if len(sys.argv) > 4 else 12
ctx = cs.shared_context(0)
w = workloads.cfg5(nq=20000)
gdb = w.build_device(ctx)
ks = np.array([len(q) for q in w.queries])
cells = np.array([math.prod(int(w.arities[v]) for v in q) for q in w.queries])
sel = np.flatnonzero((ks == k) & (cells > lo) & (cells <= hi))[:n]
qs = [w.queries[i] for i in sel]
plan = QueryPlan(gdb, qs, 1)
tabs = torch.empty(plan.total_cells, dtype=torch.int32, device="cuda")
ll = torch.empty(plan.nq, dtype=torch.float64, device="cuda")
for _ in range(2):
    plan.execute(tables=tabs, loglik=ll)
    ctx.sync()
    print("hist_ms", ctx.last_kernel_ms(), "queries", len(qs), flush=True)
