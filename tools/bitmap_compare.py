"""Bitmap class (K7, CS_BITMAP=1) vs the histogram classes (CS_BITMAP=0) on binary data.

python tools/bitmap_compare.py [m] [nq]   -> one JSON line per (k, class): device ms per batch
(CUDA events on the context stream, L2 flushed between reps), queries/s, plane / column bytes.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200.engine import GpuDatabase, QueryPlan  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
ctx = cs.shared_context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
n = 100
rng = np.random.default_rng(1)
p = rng.uniform(0.02, 0.5, n)
data = torch.from_numpy((rng.random((n, m), dtype=np.float32) < p[:, None].astype(np.float32)).astype(np.uint8)).cuda()
gdb = GpuDatabase.from_columns(ctx, data, [2] * n)
gdb.bitmap_build()
del data
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for k in (1, 2, 3, 4):
    qs = [tuple(int(x) for x in rng.choice(n, k, replace=False)) for _ in range(nq)]
    res = {}
    for mode in ("0", "1"):
        os.environ["CS_BITMAP"] = mode
        plan = QueryPlan(gdb, qs, 1)
        tabs = torch.empty(plan.total_cells, dtype=torch.int32, device="cuda")
        ll = torch.empty(nq, dtype=torch.float64, device="cuda")
        for _ in range(2):
            plan.execute(tables=tabs, loglik=ll)
        times = []
        for _ in range(5):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            plan.execute(tables=tabs, loglik=ll)
            b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b))
        res[mode] = (float(np.median(times)), tabs.cpu().numpy().copy())
        plan.close()
    same = bool(np.array_equal(res["0"][1], res["1"][1]))
    for mode, name in (("0", "histogram"), ("1", "bitmap")):
        ms = res[mode][0]
        print(json.dumps({"k": k, "class": name, "m": m, "queries": nq, "ms": round(ms, 4),
                          "queries_per_s": nq / ms * 1e3,
                          "input_gbs": nq * k * m / (8 if mode == "1" else 4) / (ms * 1e-3) / 1e9,
                          "tables_identical": same}), flush=True)
