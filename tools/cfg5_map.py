"""cfg5 (m = 1e8) roofline map: histogram-phase device time of the stream's queries grouped by
(k, table-size bucket), each group as its own plan, against the bytes of the 4-bit column copy
it reads (k * m / 2 per query) and the measured HBM peak.

    python tools/cfg5_map.py [per_group] [KNOB=value,...]
"""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200 import workloads  # noqa: E402
from paper_1804_04640_b200.engine import QueryPlan  # noqa: E402

per = int(sys.argv[1]) if len(sys.argv) > 1 else 48
for a in sys.argv[2:]:
    for kv in a.split(","):
        if kv:
            k, v = kv.split("=")
            os.environ[k] = v
peak = 6451.2
try:
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
ctx = cs.shared_context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
w = workloads.cfg5(nq=20000)
gdb = w.build_device(ctx)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
ks = np.array([len(q) for q in w.queries])
cells = np.array([math.prod(int(w.arities[v]) for v in q) for q in w.queries])
edges = [0, 41, 1760, 3520, 7040, 14080, 28160, 56320, 112640, 225280, 450560, 901120, 1 << 21, 1 << 24]
tot_t = tot_b = 0.0
KS = [int(x) for x in os.environ.get("CFG5_MAP_KS", "2,3,4,5,6,7,8").split(",")]
for k in KS:
    for lo, hi in zip(edges[:-1], edges[1:]):
        sel = np.flatnonzero((ks == k) & (cells > lo) & (cells <= hi))
        if len(sel) < 4:
            continue
        share = float(ks[sel].sum()) / float(ks.sum())
        qs = [w.queries[i] for i in sel[:per]]
        plan = QueryPlan(gdb, qs, 1)
        tabs = torch.empty(plan.total_cells, dtype=torch.int32, device="cuda")
        ll = torch.empty(plan.nq, dtype=torch.float64, device="cuda")
        plan.execute(tables=tabs, loglik=ll)
        ts = []
        for _ in range(3):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            plan.execute(tables=tabs, loglik=ll)
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        nbytes = len(qs) * k * w.m / 2
        gbs = nbytes / ms / 1e6
        tot_t += share * (ms / len(qs)) / k  # time per byte-share unit
        tot_b += share
        print(json.dumps({"k": k, "cells": [lo, hi], "n": len(qs), "byte_share": round(share, 4),
                          "us_per_query": round(ms / len(qs) * 1e3, 1), "gbs_4bit": round(gbs, 1),
                          "frac": round(gbs / peak, 3)}), flush=True)
        plan.close()
        del tabs, ll
