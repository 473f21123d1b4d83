"""Stress / parity check of cs_itemset_supports at n = 200 items and a given m (pair supports vs
a dense product).  Used to shake out pipeline races:  PYTHONPATH=. python tools/itemset_stress.py 8000000"""
import os, sys
import numpy as np
from paper_1804_04640_b200.engine import GpuContext, GpuDatabase
ctx = GpuContext(0)
rng = np.random.default_rng(5)
n = 200
m = int(sys.argv[1])
u8 = (rng.random((n, m)) < 0.3).astype(np.uint8)
g = GpuDatabase.from_columns(ctx, u8, [2] * n)
g.bitmap_build()
try:
    pr, tr = g.itemset_supports(list(range(n)))
except Exception as e:
    print("m", m, "FAIL", str(e)[:120]); sys.exit(0)
x = u8.astype(np.float32)
g2 = x @ x.T
iu = np.triu_indices(n, 1)
print("m", m, "ok", np.array_equal(pr[iu], g2[iu].astype(np.int64)))
