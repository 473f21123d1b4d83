"""Diagnostic (GPU): which cfg5 tables at full m do not sum to m, by class knobs."""
import math
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200 import workloads  # noqa: E402
from paper_1804_04640_b200._native import CS_WANT_TABLES  # noqa: E402
from paper_1804_04640_b200.engine import QueryPlan  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
ctx = cs.shared_context(0)
w = workloads.cfg5(nq=nq, m=m)
t0 = time.time()
gdb = w.build_device(ctx)
ctx.sync()
print("build", time.time() - t0, flush=True)


def sums(qs):
    plan = QueryPlan(gdb, qs, CS_WANT_TABLES)
    dev = torch.empty(plan.total_cells, dtype=torch.int32, device="cuda")
    plan.execute(tables=dev)
    ctx.sync()
    c = torch.cumsum(dev.to(torch.int64), 0).cpu().numpy()
    ends = plan.table_off + plan.cells - 1
    st = np.where(plan.table_off > 0, c[np.maximum(plan.table_off - 1, 0)], 0)
    plan.close()
    return c[ends] - st


for env in [{}, {"CS_RADIX": "0"}, {"CS_SEG_MAX_ROWS": "1048576"}]:
    for k, v in env.items():
        os.environ[k] = v
    s = sums(w.queries)
    bad = np.flatnonzero(s != m)
    cells = np.array([math.prod(int(w.arities[v]) for v in q) for q in w.queries])
    ks = np.array([len(q) for q in w.queries])
    print(env, "bad", len(bad), "of", len(s), flush=True)
    if len(bad):
        print("  bad cells range", cells[bad].min(), cells[bad].max(), "good cells range",
              cells[s == m].min() if (s == m).any() else None, cells[s == m].max() if (s == m).any() else None)
        print("  bad k hist", np.bincount(ks[bad], minlength=9).tolist(), "all", np.bincount(ks, minlength=9).tolist())
        print("  sum/m of first bad", (s[bad[:10]] / m).round(4).tolist(), "cells", cells[bad[:10]].tolist())
        # single-query plans for the first bad ones
        for i in bad[:3]:
            print("   single", i, sums([w.queries[i]])[0] / m)
    for k in env:
        del os.environ[k]
