"""Drop-in GpuStrategy.query_batch (LL only) on cfg2's workload: one-shot chunked cs_query_batch
vs an explicit QueryPlan per call (the path it used before).  Wall clock per call, host numpy
outputs, after warm-up.  Usage: python tools/dropin_batch_probe.py"""
import time
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200 import workloads  # noqa: E402
from paper_1804_04640_b200.harness import DeviceDatabase  # noqa: E402
from paper_1804_04640_b200.engine import QueryPlan  # noqa: E402

ctx = cs.shared_context(0)
w = workloads.cfg2()
gdb = w.build_device(ctx)
s = cs.GpuStrategy(DeviceDatabase(gdb), bitmaps=False)
qs = [cs.QuerySpec(q[0], tuple(q[1:])) for q in w.queries]


def plan_path():
    p = QueryPlan(gdb, [tuple(q) for q in w.queries], 0)
    ll = np.zeros(len(qs))
    p.execute(loglik=ll)
    p.close()
    return ll


def one_shot():
    return s.query_batch(qs, loglik=True)["loglik"]


off, flat = cs.encode_queries([tuple(q) for q in w.queries])


def engine_one_shot():
    ll = np.zeros(len(qs))
    gdb.query_batch(off, flat, 0, loglik=ll)
    return ll


def validate_only():
    for q in qs:
        q.validate(s.db)


for name, fn in (("QueryPlan per call", plan_path), ("engine cs_query_batch (encoded)", engine_one_shot),
                 ("GpuStrategy.query_batch (validate + encode + one-shot)", one_shot),
                 ("QuerySpec.validate x N only", validate_only)):
    for _ in range(3):
        ref = fn()
    t = []
    for _ in range(10):
        t0 = time.perf_counter()
        fn()
        t.append(time.perf_counter() - t0)
    print(f"{name}: {1e3 * np.median(t):.3f} ms per {len(qs)}-query call "
          f"({len(qs) / np.median(t) / 1e6:.2f} M q/s)")
a, b = plan_path(), one_shot()
print("max rel diff", float(np.max(np.abs(a - b) / np.abs(a))))
