"""cfg5 (m = 1e8, first N stream queries): histogram-phase device time of the same batch under
class knobs (CUDA events around plan.execute on the context stream, L2 flushed before each rep).

    python tools/cfg5_classes.py [nq] [KNOB=value,...] [KNOB=value,...] ...
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200 import workloads  # noqa: E402
from paper_1804_04640_b200.engine import QueryPlan  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
settings = [dict(kv.split("=") for kv in a.split(",") if kv) for a in sys.argv[2:]] or [{}]
ctx = cs.shared_context(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx.set_stream(stream.cuda_stream)
w = workloads.cfg5(nq=nq)
gdb = w.build_device(ctx)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
ref = None
for env in settings:
    for k, v in env.items():
        os.environ[k] = v
    bench_like = os.environ.get("CFG5_BENCH_OUTPUTS") == "1"  # bench.py's cfg5 outputs: LL + MI, no tables flag
    plan = QueryPlan(gdb, w.queries, 0 if bench_like else 1)
    tabs = torch.empty(plan.total_cells, dtype=torch.int32, device="cuda")
    ll = torch.empty(plan.nq, dtype=torch.float64, device="cuda")
    mi = torch.empty(plan.nq, dtype=torch.float64, device="cuda") if bench_like else None
    plan.execute(tables=tabs, loglik=ll, mi=mi)
    ts, ks = [], []
    for _ in range(3):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.execute(tables=tabs, loglik=ll, mi=mi)
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b))
        ks.append(ctx.last_kernel_ms())
    h = int(torch.sum(tabs.to(torch.int64) * torch.arange(1, plan.total_cells + 1, device="cuda") % 1000003).item())
    ref = h if ref is None else ref
    print(json.dumps({"env": env, "step_ms": float(np.median(ts)), "hist_ms": float(np.median(ks)),
                      "q_per_s": nq / float(np.median(ts)) * 1e3, "tables_match_first": h == ref}), flush=True)
    plan.close()
    for k in env:
        del os.environ[k]
