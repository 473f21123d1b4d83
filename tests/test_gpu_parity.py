"""GPU parity: libcountgpu (through the C ABI / drop-in Strategy) vs the pinned oracle.

Counts must be bit-exact; LL / MDL within 1e-9 relative (BASELINE north_star), MI
within the absolute bound survey 8a derives for its cancellation.
"""

from __future__ import annotations

import math
import os

import numpy as np
import pytest

import oracle as O
from conftest import FIXTURE_X1_GIVEN_X0_X2, case_db, golden_records, rel_close, sweep_db

pytestmark = pytest.mark.gpu

import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200 import workloads  # noqa: E402
from paper_1804_04640_b200.engine import GpuDatabase, QueryPlan  # noqa: E402
import gen_twin  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return cs.shared_context(0)


def _recs(result: set) -> set:
    return {(r.config, r.k, r.n_ijk, r.n_ij) for r in result}


def test_fixture_kats(reference_cases):
    db = case_db(reference_cases["fixture"])
    s = cs.GpuStrategy(db)
    col = cs.RecordCollector()
    s.query(cs.QuerySpec(1, (0, 2)), col)
    assert _recs(col.result()) == FIXTURE_X1_GIVEN_X0_X2
    col = cs.RecordCollector()
    s.query(cs.QuerySpec(1, (2, 0)), col)
    assert _recs(col.result()) == FIXTURE_X1_GIVEN_X0_X2
    assert s.count(cs.Assignment((0, 1, 2), (2, 1, 0))) == 2
    assert s.count(cs.Assignment((), ())) == 8
    sink = cs.NullSink()
    s.query(cs.QuerySpec(1, (0, 2)), sink)
    assert sink.count == 7


@pytest.mark.parametrize("name", ["fixture", "synthetic-ternary", "synthetic-binary",
                                  "synthetic-mixed-arity", "synthetic-quaternary", "synthetic-wide-binary"])
def test_reference_cases(reference_cases, name):
    case = reference_cases[name]
    db = case_db(case)
    s = cs.GpuStrategy(db)
    for q in case["queries"]:
        qs = cs.QuerySpec(q["target"], tuple(q["parents"]))
        col = cs.RecordCollector()
        s.query(qs, col)
        assert _recs(col.result()) == golden_records(q)
        ll = cs.LogLikelihood()
        s.query(qs, ll)
        assert rel_close(ll.result(), q["loglik"], 1e-9)
        assert rel_close(cs.mdl_score(db, qs, s), q["mdl"], 1e-9)
        # unfused stream path (generic aggregator) delivers the same cells
        class Tally(cs.Aggregator):
            def __init__(self):
                self.cells = []

            def accept(self, a, b):
                self.cells.append((a, b))

            def result(self):
                return self.cells

        t = Tally()
        s.query(qs, t)
        assert sorted(t.result()) == sorted((r[2], r[3]) for r in golden_records(q))
    res = cs.learn_parents(db, s, max_parents=case["learn"]["maxParents"])
    for r, want in zip(res, case["learn"]["parentSets"]):
        assert list(r.parents) == want["parents"]
        assert rel_close(r.score, want["score"], 1e-9)
    if "rules" in case:
        rr = case["rules"]
        got = cs.mine_rules(db, s, rr["minSupport"], rr["minConfidence"], rr["maxSize"])
        got = sorted(got, key=lambda r: (list(r.antecedent), r.consequent))
        assert [(list(r.antecedent), r.consequent) for r in got] == \
            [(r["antecedent"], r["consequent"]) for r in rr["rules"]]
        for a, b in zip(got, rr["rules"]):
            assert rel_close(a.support, b["support"], 1e-12) and rel_close(a.confidence, b["confidence"], 1e-12)


def test_random_sweep(random_sweep):
    for d in random_sweep["dbs"]:
        db = sweep_db(d)
        s = cs.GpuStrategy(db)
        qs = [cs.QuerySpec(q["target"], tuple(q["parents"])) for q in d["queries"]]
        out = s.query_batch(qs, loglik=True, nnz=True, tables=True)
        one_shot = s.query_batch(qs, loglik=True, mi=True, nnz=True)  # cs_query_batch path
        assert one_shot["tables"] is None and np.array_equal(one_shot["nnz"], out["nnz"])
        assert all(rel_close(a, b, 1e-12) for a, b in zip(one_shot["loglik"], out["loglik"]))
        for i, q in enumerate(d["queries"]):
            want = golden_records(q)
            c0, c1 = out["table_off"][i], out["table_off"][i] + out["cells"][i]
            got = O.records_from_table(out["tables"][c0:c1], q["target"], q["parents"], db.arities)
            assert got == want
            assert out["nnz"][i] == len(want)
            assert rel_close(out["loglik"][i], q["loglik"], 1e-9)
            col = cs.RecordCollector()
            s.query(qs[i], col)
            assert _recs(col.result()) == want
        counts = s.count_batch([cs.Assignment(p["vars"], p["states"]) for p in d["points"]])
        assert counts.tolist() == [p["count"] for p in d["points"]]


def test_point_counts_scan_and_bitmap_paths(random_sweep):
    for d in random_sweep["dbs"][:20]:
        db = sweep_db(d)
        g_scan = cs.GpuStrategy(db, bitmaps=False)
        g_bits = cs.GpuStrategy(db, bitmaps=True)
        al = [cs.Assignment(p["vars"], p["states"]) for p in d["points"]]
        want = [p["count"] for p in d["points"]]
        assert g_scan.count_batch(al).tolist() == want
        assert g_bits.count_batch(al).tolist() == want


def test_cfg1_bit_exact(ctx, cfg1_golden):
    g = cfg1_golden
    w = workloads.cfg1(int(g["seed"]))
    assert np.array_equal(w.host_db.columns_u8(), g["data"])
    gdb = w.build_device(ctx)
    plan = QueryPlan(gdb, [tuple(q) for q in g["queries"]], cs._native.CS_WANT_TABLES)
    tabs = np.zeros(plan.total_cells, dtype=np.uint32)
    ll = np.zeros(plan.nq)
    plan.execute(tables=tabs, loglik=ll)
    assert np.array_equal(plan.table_off, g["table_off"])
    assert np.array_equal(tabs, g["tables"])
    assert np.allclose(ll, g["loglik"], rtol=1e-9, atol=1e-12)


def _check_plan_vs_oracle(gdb, cols_u8, arities, queries, rtol=1e-9):
    plan = QueryPlan(gdb, queries, cs._native.CS_WANT_TABLES)
    tabs = np.zeros(plan.total_cells, dtype=np.uint32)
    ll = np.zeros(plan.nq)
    nnz = np.zeros(plan.nq, dtype=np.int64)
    plan.execute(tables=tabs, loglik=ll, nnz=nnz)
    otabs, ooff, oll, onnz = O.radix_tables(cols_u8, arities, queries)
    assert np.array_equal(plan.table_off, ooff)
    assert np.array_equal(tabs, otabs)
    assert np.array_equal(nnz, onnz)
    assert np.allclose(ll, oll, rtol=rtol, atol=1e-12)
    return plan, tabs


def test_generator_twin_and_cfg2_slice(ctx):
    w = workloads.cfg2(nq=300, m=200_003)
    gdb = w.build_device(ctx)
    rows = np.arange(w.m)
    cols = gen_twin.generate_workload_columns(w, rows)
    u8 = np.vstack([cols[v] for v in range(w.n)])
    for v in range(0, w.n, 7):
        assert np.array_equal(gdb.download(v), u8[v])
    _check_plan_vs_oracle(gdb, u8, w.arities, w.queries)


def test_cfg3_slice_and_learning(ctx):
    w = workloads.cfg3(m=50_000, n=12)
    gdb = w.build_device(ctx)
    cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
    u8 = np.vstack([cols[v] for v in range(w.n)])
    assert np.array_equal(gdb.download(w.n - 1), u8[w.n - 1])
    _check_plan_vs_oracle(gdb, u8, w.arities, w.queries[:2000])


@pytest.mark.parametrize("env", [{"CS_SEG_MAX_ROWS": "65536"}, {"CS_HIST_SMEM_KB": "8"}])
def test_multisegment_and_global_classes(env):
    """Force the multi-segment merge (last-CTA scoring) and the global-atomic class."""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        c = cs.GpuContext(0)
        w = workloads.cfg2(nq=120, m=400_000, seed=11)
        gdb = w.build_device(c)
        cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
        u8 = np.vstack([cols[v] for v in range(w.n)])
        _check_plan_vs_oracle(gdb, u8, w.arities, w.queries)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _big_table_workload(m, nq=24, seed=7):
    """cfg5-shaped data (arity U{2..8}) with only tables above SMEM capacity (56K..2^24 cells)."""
    w = workloads.cfg5(seed=seed, nq=4000, m=m, n=40)
    qs = [q for q in w.queries if np.prod([int(w.arities[v]) for v in q]) > 60_000][:nq]
    return w, qs


@pytest.mark.parametrize("env", [{}, {"CS_SPILL": "0"}, {"CS_SPILL": "0", "CS_RADIX_CPI": "2", "CS_RADIX_MB": "1"},
                                 {"CS_SPILL": "0", "CS_RADIX": "0"}])
def test_partition_class_big_tables(env):
    """Tables above SMEM capacity: the partition class (one counting-sort pass + SMEM group
    histograms), forced into many count items / one-query waves, and the slice / global
    classes it replaces (CS_RADIX=0) -- bit-exact tables, LL and nnz vs the radix oracle.
    m is not a multiple of the 32-row vector or the 16K-row chunk."""
    def run():
        c = cs.GpuContext(0)
        w, qs = _big_table_workload(m=70_001)
        gdb = w.build_device(c)
        cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
        u8 = np.vstack([cols[v] for v in range(w.n)])
        _check_plan_vs_oracle(gdb, u8, w.arities, qs)
    _with_env(env, run)


def test_partition_class_tiny_m(ctx):
    """Fewer rows than one partition chunk, and a database of 1 row."""
    for m in (1, 33, 5_000):
        w, qs = _big_table_workload(m=m, nq=6, seed=9)
        gdb = w.build_device(ctx)
        cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
        u8 = np.vstack([cols[v] for v in range(w.n)])
        _check_plan_vs_oracle(gdb, u8, w.arities, qs)


def test_partition_class_mi_and_records(ctx):
    """Fused MI through the chunked scorer and the record stream of a partition-class table."""
    w, qs = _big_table_workload(m=40_000, nq=4, seed=13)
    gdb = w.build_device(ctx)
    cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
    u8 = np.vstack([cols[v] for v in range(w.n)])
    plan = QueryPlan(gdb, qs)
    mi = np.zeros(plan.nq)
    ll = np.zeros(plan.nq)
    plan.execute(loglik=ll, mi=mi)
    for i, q in enumerate(qs):
        recs = O.oracle_records(u8, w.arities, q[0], q[1:])
        ll1 = O.loglik_of_records(recs)
        ll0 = O.loglik_of_records(O.oracle_records(u8, w.arities, q[0], ()))
        assert rel_close(ll[i], ll1, 1e-9)
        assert abs(mi[i] - O.mi_of_records(recs, w.m)) <= 1e-9 * (abs(ll1) + abs(ll0)) / w.m


def test_generic_many_variable_queries(ctx):
    rng = np.random.default_rng(5)
    n, m = 14, 3001
    ar = rng.integers(2, 4, size=n)
    u8 = np.vstack([rng.integers(0, r, m) for r in ar]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, u8, ar)
    qs = [tuple(int(x) for x in rng.choice(n, size=k, replace=False)) for k in (9, 10, 11, 12) for _ in range(3)]
    _check_plan_vs_oracle(gdb, u8, ar, qs)


def test_mi_fused(ctx):
    w = workloads.cfg2(nq=200, m=100_000, seed=3)
    gdb = w.build_device(ctx)
    cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
    u8 = np.vstack([cols[v] for v in range(w.n)])
    qs = [q for q in w.queries if len(q) >= 2][:60]
    plan = QueryPlan(gdb, qs)
    mi = np.zeros(plan.nq)
    ll = np.zeros(plan.nq)
    plan.execute(loglik=ll, mi=mi)
    for i, q in enumerate(qs):
        recs = O.oracle_records(u8, w.arities, q[0], q[1:])
        want = O.mi_of_records(recs, w.m)
        ll1 = O.loglik_of_records(recs)
        ll0 = O.loglik_of_records(O.oracle_records(u8, w.arities, q[0], ()))
        tol = 1e-9 * (abs(ll1) + abs(ll0)) / w.m
        assert abs(mi[i] - want) <= tol, (q, mi[i], want)


def test_properties_full_size(ctx):
    """At full cfg2 size: every table sums to m, and marginalising a table over its last
    parent equals the table of the shorter query (size-independent properties)."""
    w = workloads.cfg2(nq=400)
    gdb = w.build_device(ctx)
    qs = [q for q in w.queries if len(q) >= 2][:200]
    shorter = [q[:-1] for q in qs]
    plan = QueryPlan(gdb, qs + shorter, cs._native.CS_WANT_TABLES)
    tabs = np.zeros(plan.total_cells, dtype=np.uint32)
    plan.execute(tables=tabs)
    for i in range(len(qs)):
        t = tabs[plan.table_off[i]:plan.table_off[i] + plan.cells[i]].astype(np.int64)
        assert int(t.sum()) == w.m
        j = i + len(qs)
        s = tabs[plan.table_off[j]:plan.table_off[j] + plan.cells[j]].astype(np.int64)
        last = int(w.arities[qs[i][-1]])
        assert np.array_equal(t.reshape(last, -1).sum(axis=0), s)


@pytest.fixture(params=["0", "1"], ids=["bitgemm", "selector"])
def itemset_path(request, monkeypatch):
    """Force the dense bit-GEMM classes (K4b/K4c) or the rarest-item selector class (K4d)."""
    monkeypatch.setenv("CS_ITEMSETS_SEL", request.param)
    return request.param


def test_itemset_supports_all_pairs_triples(ctx, itemset_path):
    """cs_itemset_supports (both classes) vs the bitmap_count restatement."""
    import itertools

    rng = np.random.default_rng(17)
    n_items, m = 45, 100_003
    p = np.clip(0.6 * np.arange(1, n_items + 1) ** -0.7, 0.01, 1.0)
    u8 = (rng.random((n_items, m)) < p[:, None]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, u8, [2] * n_items)
    gdb.bitmap_build()
    items = list(range(3, n_items))  # a subset, not starting at 0
    pr, tr = gdb.itemset_supports(items)
    planes = {(v, 1): O.bitmap_planes(u8[v], 1) for v in items}
    pairs = list(itertools.combinations(range(len(items)), 2))
    want_p = O.bitmap_counts(planes, [((items[a], 1), (items[b], 1)) for a, b in pairs], m)
    assert [int(pr[a, b]) for a, b in pairs] == want_p.tolist()
    triples = list(itertools.combinations(range(len(items)), 3))
    want_t = O.bitmap_counts(planes, [tuple((items[x], 1) for x in t) for t in triples], m)
    assert np.array_equal(tr, want_t)
    # point-count path agrees on a sample
    sample = triples[::97]
    got = gdb.count_points([([items[x] for x in t], [1, 1, 1]) for t in sample])
    assert got.tolist() == [int(want_t[triples.index(t)]) for t in sample]


def test_itemset_supports_wide_chunked(ctx):
    """> 256 items: several tensor-core column chunks per row block; ragged m (not a multiple of
    the 256-row step).  Checked against dense products for a sample of first items a."""
    rng = np.random.default_rng(23)
    n, m = 300, 20_011
    p = np.clip(0.7 * np.arange(1, n + 1) ** -0.3, 0.02, 1.0)
    u8 = (rng.random((n, m)) < rng.permutation(p)[:, None]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, u8, [2] * n)
    gdb.bitmap_build()
    pr, tr = gdb.itemset_supports(list(range(n)))
    x = u8.astype(np.float64)
    g2 = x @ x.T
    iu = np.triu_indices(n, 1)
    assert np.array_equal(pr[iu], g2[iu].astype(np.int64))

    def c3(v):
        return v * (v - 1) * (v - 2) // 6 if v >= 3 else 0

    def c2(v):
        return v * (v - 1) // 2 if v >= 2 else 0

    for a in (0, 1, 77, 128, 255, 256, 297):
        t = (x * x[a]) @ x.T  # t[b, c] = support(a, b, c)
        for b in range(a + 1, n - 1):
            base = c3(n) - c3(n - a) + c2(n - a - 1) - c2(n - b)
            got = tr[base:base + (n - b - 1)]
            assert np.array_equal(got, t[b, b + 1:].astype(np.int64)), (a, b)


def test_cfg4_workload_small(ctx, itemset_path):
    """configs[3] generator + top-k selection + supports at reduced m."""
    w = workloads.cfg4(m=200_000, n_items=300, top=40)
    gdb = w.build_device(ctx)
    sup = gdb.count_points([((v,), (1,)) for v in range(w.n)])
    rows = np.arange(w.m)
    cols = gen_twin.generate_workload_columns(w, rows)
    assert sup.tolist() == [int(cols[v].sum()) for v in range(w.n)]
    top = workloads.select_top_items(sup, 40)
    gdb.bitmap_build(top)
    pr, tr = gdb.itemset_supports(top)
    planes = {(v, 1): O.bitmap_planes(cols[v], 1) for v in top}
    its = workloads.itemsets_of(range(len(top)), (3,))
    want = O.bitmap_counts(planes, [tuple((top[x], 1) for x in t) for t in its], w.m)
    assert np.array_equal(tr, want)


def test_family_scores_match_per_query(ctx):
    """Subset N ln N differences reproduce per-family LL / MDL (cfg3-shaped, reduced)."""
    from paper_1804_04640_b200.engine import FamilyScorer

    w = workloads.cfg3(m=60_000, n=10)
    gdb = w.build_device(ctx)
    cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
    u8 = np.vstack([cols[v] for v in range(w.n)])
    fams = [(q[0], tuple(q[1:])) for q in w.queries]
    fs = FamilyScorer(gdb, fams)
    ll, mdl = fs.scores()
    _, _, oll, _ = O.radix_tables(u8, w.arities, w.queries, want_tables=False)
    assert np.allclose(ll, oll, rtol=1e-9, atol=1e-9)
    for f, (t, ps) in enumerate(fams[:500]):
        q_i = int(np.prod([int(w.arities[p]) for p in ps])) if ps else 1
        assert rel_close(mdl[f], O.mdl_of(oll[f], w.m, int(w.arities[t]), q_i), 1e-9)


def test_duck_typed_reference_objects(reference_cases):
    """The drop-in accepts reference-style query/aggregator objects it did not define."""
    import types

    db = case_db(reference_cases["fixture"])
    s = cs.GpuStrategy(db)

    class RefQuery:  # the reference QuerySpec surface: target, parents, validate(db)
        def __init__(self, target, parents):
            self.target, self.parents = target, tuple(parents)

        def validate(self, db):
            pass

    # a LogLikelihood-shaped object from the reference module is fused by type name
    RefLL = type("LogLikelihood", (), {"__module__": "countstream.aggregators", "wants_records": False,
                                       "__init__": lambda self: setattr(self, "total", 0.0)})
    agg = RefLL()
    s.query(RefQuery(1, (0, 2)), agg)
    want = O.loglik_of_records(FIXTURE_X1_GIVEN_X0_X2)
    assert rel_close(agg.total, want, 1e-12)
    col = cs.RecordCollector()
    s.query(RefQuery(1, (2, 0)), col)
    assert _recs(col.result()) == FIXTURE_X1_GIVEN_X0_X2


@pytest.mark.parametrize("smem_kb", ["220", "8"])
def test_instance_sharded_merge_on_one_gpu(smem_kb):
    """CS_PARTIAL tables of two row shards, summed on the device, then cs_plan_score with the
    global m (the cfg5 NCCL path minus the collective) == oracle LL / MI on the full data.
    smem_kb=8 forces the global-atomic class and the chunked K2 scorer."""
    import torch

    old = os.environ.get("CS_HIST_SMEM_KB")
    os.environ["CS_HIST_SMEM_KB"] = smem_kb
    try:
        c = cs.GpuContext(0)
        w = workloads.cfg5(nq=40, m=300_001, n=30, seed=7)
        cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
        u8 = np.vstack([cols[v] for v in range(w.n)])
        from paper_1804_04640_b200.parallel import shard_rows

        parts = []
        for r in range(2):
            r0, nr = shard_rows(w.m, 2, r)
            g = w.build_device(c, row_offset=r0, m_shard=nr)
            assert np.array_equal(g.download(3), u8[3, r0:r0 + nr])
            plan = QueryPlan(g, w.queries, cs._native.CS_PARTIAL | cs._native.CS_WANT_TABLES)
            t = torch.zeros(plan.total_cells, dtype=torch.int32, device="cuda")
            plan.execute(tables=t)
            parts.append((g, plan, t))
        c.sync()  # device outputs are asynchronous on the context stream
        merged = parts[0][2] + parts[1][2]
        torch.cuda.synchronize()
        plan = parts[1][1]
        ll = torch.zeros(plan.nq, dtype=torch.float64, device="cuda")
        mi = torch.zeros(plan.nq, dtype=torch.float64, device="cuda")
        nnz = torch.zeros(plan.nq, dtype=torch.int64, device="cuda")
        plan.score(merged, loglik=ll, mi=mi, nnz=nnz)
        c.sync()
        otabs, _, oll, onnz = O.radix_tables(u8, w.arities, w.queries)
        assert np.array_equal(merged.cpu().numpy().view(np.uint32), otabs)
        assert np.allclose(ll.cpu().numpy(), oll, rtol=1e-9, atol=1e-9)
        assert np.array_equal(nnz.cpu().numpy(), onnz)
        for i, q in enumerate(w.queries[:25]):
            recs = O.oracle_records(u8, w.arities, q[0], q[1:])
            ll0 = O.loglik_of_records(O.oracle_records(u8, w.arities, q[0], ()))
            tol = 1e-9 * (abs(oll[i]) + abs(ll0)) / w.m
            assert abs(mi[i].item() - O.mi_of_records(recs, w.m)) <= tol
    finally:
        if old is None:
            os.environ.pop("CS_HIST_SMEM_KB", None)
        else:
            os.environ["CS_HIST_SMEM_KB"] = old


def test_sparse_hash_class(random_sweep):
    """Joint state spaces beyond the dense limit go to the hash class: forced with a tiny dense
    limit on the random sweep, plus a genuine 2^40-cell query (40 binary variables)."""
    old = os.environ.get("CS_MAX_DENSE_LOG2")
    os.environ["CS_MAX_DENSE_LOG2"] = "6"
    try:
        for d in random_sweep["dbs"][:25]:
            db = sweep_db(d)
            s = cs.GpuStrategy(db)
            for q in d["queries"]:
                qs = cs.QuerySpec(q["target"], tuple(q["parents"]))
                col = cs.RecordCollector()
                s.query(qs, col)
                assert _recs(col.result()) == golden_records(q)
                ll = cs.LogLikelihood()
                s.query(qs, ll)
                assert rel_close(ll.result(), q["loglik"], 1e-9)
                sink = cs.NullSink()
                s.query(qs, sink)
                assert sink.count == len(q["records"])
    finally:
        if old is None:
            os.environ.pop("CS_MAX_DENSE_LOG2", None)
        else:
            os.environ["CS_MAX_DENSE_LOG2"] = old
    rng = np.random.default_rng(3)
    data = (rng.random((40, 5000)) < rng.uniform(0.2, 0.8, size=(40, 1))).astype(np.int32)
    db = cs.Database(data, [2] * 40)
    s = cs.GpuStrategy(db)
    qs = cs.QuerySpec(0, tuple(range(1, 40)))
    col = cs.RecordCollector()
    s.query(qs, col)
    want = O.oracle_records(data, db.arities, 0, tuple(range(1, 40)))
    assert _recs(col.result()) == want
    ll = cs.LogLikelihood()
    s.query(qs, ll)
    assert rel_close(ll.result(), O.loglik_of_records(want), 1e-9)
    mi = cs.MutualInformation(db.m)
    s.query(qs, mi)
    assert abs(mi.result() - O.mi_of_records(want, db.m)) < 1e-9


def test_cfg2_full_size_sample(ctx):
    """configs[1] at full size (m = 1e6): a 200-query sample, bit-exact against the radix
    restatement on the twin-regenerated columns."""
    w = workloads.cfg2()
    gdb = w.build_device(ctx)
    qs = w.queries[:200]
    vs = sorted({v for q in qs for v in q})
    cols = gen_twin.generate_workload_columns(w, np.arange(w.m), vs)
    remap = {v: i for i, v in enumerate(vs)}
    u8 = np.vstack([cols[v] for v in vs])
    plan = QueryPlan(gdb, qs, cs._native.CS_WANT_TABLES)
    tabs = np.zeros(plan.total_cells, dtype=np.uint32)
    ll = np.zeros(plan.nq)
    plan.execute(tables=tabs, loglik=ll)
    otabs, ooff, oll, _ = O.radix_tables(u8, w.arities[vs], [tuple(remap[v] for v in q) for q in qs])
    assert np.array_equal(tabs, otabs)
    assert np.allclose(ll, oll, rtol=1e-9, atol=1e-9)


def test_cfg4_full_m_sample(ctx, itemset_path):
    """configs[3] at full m = 1e7: supports of all pairs/triples of 10 of the top items vs the
    bitmap_count restatement on twin-regenerated columns."""
    w = workloads.cfg4()
    gdb = w.build_device(ctx)
    sup = gdb.count_points([((v,), (1,)) for v in range(w.n)])
    top = workloads.select_top_items(sup, 200)
    sample = top[::20]  # 10 items spread over the frequency range
    gdb.bitmap_build(sample)
    pr, tr = gdb.itemset_supports(sample)
    cols = gen_twin.generate_workload_columns(w, np.arange(w.m), sample)
    assert [int(sup[v]) for v in sample] == [int(cols[v].sum()) for v in sample]
    planes = {(v, 1): O.bitmap_planes(cols[v], 1) for v in sample}
    import itertools

    tri = list(itertools.combinations(range(len(sample)), 3))
    want = O.bitmap_counts(planes, [tuple((sample[x], 1) for x in t) for t in tri], w.m)
    assert np.array_equal(tr, want)
    pairs = list(itertools.combinations(range(len(sample)), 2))
    wantp = O.bitmap_counts(planes, [((sample[a], 1), (sample[b], 1)) for a, b in pairs], w.m)
    assert [int(pr[a, b]) for a, b in pairs] == wantp.tolist()


def test_cfg4_full_classes_agree(ctx, monkeypatch):
    """configs[3] in full (200 items, m = 1e7): the selector class (the bench path) and the
    tensor-core bit-GEMM give identical pair and triple supports, and a spread of 12 items'
    pairs/triples (indexed inside the 200-item numbering) match bitmap_count on twin columns."""
    import itertools

    w = workloads.cfg4()
    gdb = w.build_device(ctx)
    sup = gdb.count_points([((v,), (1,)) for v in range(w.n)])
    top = workloads.select_top_items(sup, 200)
    gdb.bitmap_build(top)
    monkeypatch.setenv("CS_ITEMSETS_SEL", "1")
    pr1, tr1 = gdb.itemset_supports(top)
    monkeypatch.setenv("CS_ITEMSETS_SEL", "0")
    pr0, tr0 = gdb.itemset_supports(top)
    assert np.array_equal(np.triu(pr1, 1), np.triu(pr0, 1))
    assert np.array_equal(tr1, tr0)
    pick = list(range(0, 200, 17))
    vars_ = [top[i] for i in pick]
    cols = gen_twin.generate_workload_columns(w, np.arange(w.m), vars_)
    planes = {(v, 1): O.bitmap_planes(cols[v], 1) for v in vars_}
    n = 200

    def tri_index(a, b, c):
        c3 = lambda v: v * (v - 1) * (v - 2) // 6 if v >= 3 else 0  # noqa: E731
        c2 = lambda v: v * (v - 1) // 2 if v >= 2 else 0  # noqa: E731
        return c3(n) - c3(n - a) + c2(n - a - 1) - c2(n - b) + (c - b - 1)

    tri = list(itertools.combinations(pick, 3))
    want = O.bitmap_counts(planes, [tuple((top[x], 1) for x in t) for t in tri], w.m)
    assert [int(tr1[tri_index(*t)]) for t in tri] == want.tolist()
    pairs = list(itertools.combinations(pick, 2))
    wantp = O.bitmap_counts(planes, [((top[a], 1), (top[b], 1)) for a, b in pairs], w.m)
    assert [int(pr1[a, b]) for a, b in pairs] == wantp.tolist()


@pytest.mark.parametrize("shape", ["two_items", "three_items", "zero_and_full", "duplicates"])
def test_itemset_supports_edges(ctx, itemset_path, shape):
    """Edge cases of cs_itemset_supports in both classes: n = 2 (no triples) and n = 3,
    items that never / always occur (ties in the support ranking), an item listed twice, and
    a row count that is not a multiple of 32."""
    import itertools

    rng = np.random.default_rng(5)
    m = 70_001
    n_items = 12
    u8 = (rng.random((n_items, m)) < np.linspace(0.02, 0.6, n_items)[:, None]).astype(np.uint8)
    u8[3] = 0  # never occurs
    u8[7] = 1  # always occurs
    u8[8] = u8[2]  # identical supports (tie)
    gdb = GpuDatabase.from_columns(ctx, u8, [2] * n_items)
    gdb.bitmap_build()
    items = {"two_items": [5, 1], "three_items": [7, 3, 4],
             "zero_and_full": list(range(n_items)), "duplicates": [2, 5, 2, 9, 7, 8]}[shape]
    pr, tr = gdb.itemset_supports(items)
    x = u8.astype(np.int64)
    for a, b in itertools.combinations(range(len(items)), 2):
        assert int(pr[a, b]) == int((x[items[a]] & x[items[b]]).sum()), (a, b)
    tri = list(itertools.combinations(range(len(items)), 3))
    assert len(tr) == len(tri)
    for i, (a, b, c) in enumerate(tri):
        assert int(tr[i]) == int((x[items[a]] & x[items[b]] & x[items[c]]).sum()), (a, b, c)


def test_pinned_host_tables_written_in_place(ctx):
    """Page-locked host tables are written by the K1 epilogues directly (zero-copy path) and
    must equal the device-table result and the oracle; pageable ones go through scratch + D2H."""
    import torch

    w = workloads.cfg2(nq=400, m=50_000)
    gdb = w.build_device(ctx)
    plan = QueryPlan(gdb, w.queries, cs._native.CS_WANT_TABLES)
    dev = torch.zeros(plan.total_cells, dtype=torch.int32, device="cuda")
    plan.execute(tables=dev)
    pinned = torch.zeros(plan.total_cells, dtype=torch.int32).pin_memory()
    plan.execute(tables=pinned)
    pageable = np.zeros(plan.total_cells, dtype=np.uint32)
    plan.execute(tables=pageable)
    d = dev.cpu().numpy().view(np.uint32)
    assert np.array_equal(pinned.numpy().view(np.uint32), d)
    assert np.array_equal(pageable, d)
    cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
    otabs, _, _, _ = O.radix_tables(np.stack([cols[v] for v in range(w.n)]), w.arities, w.queries)
    assert np.array_equal(d, otabs)


def test_plan_threads_identical(ctx, monkeypatch):
    """A 6,000-query mixed batch (SMEM, packed, radix, slice, generic > 8 variables and hash
    classes) planned serially and on 8 host threads gives identical tables and scores; a bad
    query deep in the batch is reported by its own index either way."""
    rng = np.random.default_rng(31)
    n, m = 40, 30_000
    ar = np.concatenate([np.full(12, 2), rng.integers(3, 9, size=14), np.full(14, 8)])
    u8 = np.stack([rng.integers(0, a, size=m) for a in ar]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, u8, ar)
    qs = []
    for i in range(6000):
        if i % 997 == 0:  # 14 variables of arity 8: 8^14 > 2^30 cells, hash class
            qs.append(tuple(int(v) for v in rng.permutation(np.arange(26, 40))))
        elif i % 50 == 0:  # 9 or 10 binary variables: generic class (> 8 digits)
            qs.append(tuple(int(v) for v in rng.choice(12, size=int(rng.integers(9, 11)), replace=False)))
        else:
            qs.append(tuple(int(v) for v in rng.choice(n, size=int(rng.integers(1, 7)), replace=False)))
    flags = cs._native.CS_WANT_TABLES
    out = []
    for threads in ("1", "8"):
        monkeypatch.setenv("CS_PLAN_THREADS", threads)
        plan = QueryPlan(gdb, qs, flags)
        tabs = np.zeros(plan.total_cells, dtype=np.uint32)
        ll = np.zeros(plan.nq)
        nnz = np.zeros(plan.nq, dtype=np.int64)
        plan.execute(tables=tabs, loglik=ll, nnz=nnz)
        out.append((tabs, ll, nnz, np.asarray(plan.table_off).copy()))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1], out[1][1])
    assert np.array_equal(out[0][2], out[1][2])
    assert np.array_equal(out[0][3], out[1][3])
    bad = list(qs)
    bad[4321] = (3, 3)
    bad[5000] = (n + 5,)
    for threads in ("1", "8"):
        monkeypatch.setenv("CS_PLAN_THREADS", threads)
        with pytest.raises(cs.InvalidQueryError, match="query 4321 repeats variable 3"):
            QueryPlan(gdb, bad, flags)


def test_pipelined_instance_sharded_single_rank(ctx):
    """The pipelined instance-sharded runner (partial tables, async NCCL all-reduce overlapped
    with the next slice's scan, per-slice scoring) on a one-rank NCCL group equals the plain
    plan's fused LL / MI."""
    import torch
    import torch.distributed as dist

    from paper_1804_04640_b200.parallel import PipelinedInstanceSharded

    w = workloads.cfg2(nq=300, m=40_000)
    gdb = w.build_device(ctx)
    own = not dist.is_initialized()
    if own:
        dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29533", rank=0, world_size=1)
    s = torch.cuda.Stream()
    ctx.set_stream(s.cuda_stream)  # library kernels and NCCL ordered on one stream
    try:
        with torch.cuda.stream(s):
            ll = torch.zeros(len(w.queries), dtype=torch.float64, device="cuda")
            mi = torch.zeros_like(ll)
            PipelinedInstanceSharded(gdb, w.queries, nbatch=4).run(loglik=ll, mi=mi)
        torch.cuda.synchronize()
    finally:
        ctx.set_stream(None)  # back to a library-owned stream
        if own:
            dist.destroy_process_group()
    plan = QueryPlan(gdb, w.queries, 0)
    ll0 = np.zeros(plan.nq)
    mi0 = np.zeros(plan.nq)
    plan.execute(loglik=ll0, mi=mi0)
    assert np.allclose(ll.cpu().numpy(), ll0, rtol=1e-12, atol=1e-9)
    assert np.allclose(mi.cpu().numpy(), mi0, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("shape", ["one_row", "one_variable", "constant_columns", "arity_256",
                                   "ragged_m_2bit", "ragged_m_4bit", "ragged_m_u8"])
def test_edge_databases(ctx, shape):
    """Degenerate databases through the counting plan vs the radix restatement (tables bit-exact,
    LL to 1e-9): a single record, a single variable (target-only queries), arity-1 (constant)
    variables, the maximum arity 256, and row counts that are not multiples of the 16/32/64-row
    vectors of the uint8 / 4-bit / 2-bit layouts.  Also an empty batch."""
    rng = np.random.default_rng(sum(shape.encode()))
    if shape == "one_row":
        ar = np.array([3, 2, 4, 2]); m = 1
    elif shape == "one_variable":
        ar = np.array([5]); m = 1_001
    elif shape == "constant_columns":
        ar = np.array([1, 3, 1, 2, 4]); m = 5_003
    elif shape == "arity_256":
        ar = np.array([256, 2, 3, 256]); m = 70_001
    elif shape == "ragged_m_2bit":
        ar = np.array([2, 3, 4, 4, 2, 3]); m = 100_003
    elif shape == "ragged_m_4bit":
        ar = np.array([2, 7, 16, 5, 3, 9]); m = 100_007
    else:
        ar = np.array([2, 17, 30, 5, 3, 9]); m = 100_011
    u8 = np.stack([rng.integers(0, a, size=m) for a in ar]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, u8, ar)
    n = len(ar)
    qs = [(v,) for v in range(n)]
    if n > 1:
        qs += [tuple(int(x) for x in rng.permutation(n)[:k]) for k in range(2, min(n, 4) + 1) for _ in range(3)]
    plan = QueryPlan(gdb, qs, cs._native.CS_WANT_TABLES)
    tabs = np.zeros(plan.total_cells, dtype=np.uint32)
    ll = np.zeros(plan.nq)
    plan.execute(tables=tabs, loglik=ll)
    otabs, _, oll, _ = O.radix_tables(u8, ar, qs)
    assert np.array_equal(tabs, otabs)
    assert np.allclose(ll, oll, rtol=1e-9, atol=1e-9)
    empty = QueryPlan(gdb, [], cs._native.CS_WANT_TABLES)
    assert empty.nq == 0 and empty.total_cells == 0
    empty.execute(tables=np.zeros(1, dtype=np.uint32), loglik=np.zeros(1))


@pytest.mark.parametrize("outputs", ["pageable", "pinned", "device"])
def test_query_batch_pipelined_chunks(ctx, outputs, monkeypatch):
    """cs_query_batch over >= CS_QB_PIPE_MIN queries plans chunk j+1 while chunk j runs (two
    scratch banks, deferred syncs): tables / LL / MI / nnz bit-identical to the one-plan path
    and to the oracle's radix restatement."""
    import torch

    rng = np.random.default_rng(1804)
    n, m = 24, 150_000
    arities = rng.integers(2, 6, size=n).astype(np.int32)
    cols = np.stack([rng.integers(0, a, size=m) for a in arities]).astype(np.uint8)
    queries = [tuple(int(v) for v in rng.choice(n, size=int(rng.integers(1, 5)), replace=False))
               for _ in range(5000)]
    gdb = GpuDatabase.from_columns(ctx, cols, arities)
    from paper_1804_04640_b200.engine import encode_queries

    off, flat = encode_queries(queries)
    cells = np.array([int(np.prod([int(arities[v]) for v in q])) for q in queries], dtype=np.int64)
    total = int(cells.sum())
    flags = cs._native.CS_WANT_TABLES

    def run(chunks):
        if chunks:
            monkeypatch.setenv("CS_QB_CHUNKS", str(chunks))
        if outputs == "device":
            mk = lambda k, dt: torch.zeros(k, dtype=dt, device="cuda")  # noqa: E731
        elif outputs == "pinned":
            mk = lambda k, dt: torch.zeros(k, dtype=dt).pin_memory()  # noqa: E731
        else:
            mk = lambda k, dt: torch.zeros(k, dtype=dt)  # noqa: E731
        t, ll, mi, nz = (mk(total, torch.int32), mk(len(queries), torch.float64),
                         mk(len(queries), torch.float64), mk(len(queries), torch.int64))
        gdb.query_batch(off, flat, flags, tables=t, loglik=ll, mi=mi, nnz=nz)
        torch.cuda.synchronize()
        return [x.cpu().numpy() for x in (t, ll, mi, nz)]

    one = run(1)
    for chunks, growth in ((2, 4), (3, 2), (5, 3)):
        monkeypatch.setenv("CS_QB_GROWTH", str(growth))
        got = run(chunks)
        # counts bit-exact; the fp64 scores' summation order follows each chunk's row segmentation
        assert np.array_equal(one[0], got[0]) and np.array_equal(one[3], got[3]), chunks
        assert all(rel_close(a, b, 1e-12) for a, b in zip(one[1], got[1])), chunks
        assert all(rel_close(a, b, 1e-12) or abs(a - b) < 1e-12 for a, b in zip(one[2], got[2])), chunks
    monkeypatch.delenv("CS_QB_CHUNKS")
    monkeypatch.delenv("CS_QB_GROWTH")
    monkeypatch.setenv("CS_QB_MIN_CHUNK", "200")  # automatic split: 5000 queries -> 3 chunks
    auto = run(0)
    assert np.array_equal(one[0], auto[0]) and np.array_equal(one[3], auto[3])
    otabs, _, oll, onnz = O.radix_tables(cols, arities, queries)
    assert np.array_equal(one[0].view(np.uint32), otabs)
    assert np.array_equal(one[3], onnz)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(one[1], oll))


@pytest.mark.parametrize("chunks", [1, 3])
def test_query_batch_score_only_chunks(ctx, chunks, monkeypatch):
    """The score-only one-shot path (no tables): one plan and forced chunking, raw C ABI and the
    drop-in GpuStrategy.query_batch with and without tables, against the dense oracle."""
    from paper_1804_04640_b200.database import Database, QuerySpec
    from paper_1804_04640_b200.engine import encode_queries
    from paper_1804_04640_b200.harness import GpuStrategy

    rng = np.random.default_rng(77)
    n, m = 16, 90_001
    arities = rng.integers(2, 6, size=n).astype(np.int32)
    cols = np.stack([rng.integers(0, a, size=m) for a in arities]).astype(np.uint8)
    queries = [tuple(int(v) for v in rng.choice(n, size=int(rng.integers(1, 6)), replace=False))
               for _ in range(3000)]
    monkeypatch.setenv("CS_QB_CHUNKS", str(chunks))
    monkeypatch.setenv("CS_QB_SCORE_MIN", "1")
    gdb = GpuDatabase.from_columns(ctx, cols, arities)
    off, flat = encode_queries(queries)
    ll, mi, nz = np.zeros(len(queries)), np.zeros(len(queries)), np.zeros(len(queries), dtype=np.int64)
    gdb.query_batch(off, flat, 0, loglik=ll, mi=mi, nnz=nz)
    _, _, oll, omi, onnz = O.dense_tables(cols, arities, queries, want_tables=False)
    assert np.array_equal(nz, onnz)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(ll, oll))
    assert np.all(np.abs(mi - omi) <= 1e-9 * (np.abs(oll) + 1) / m + 1e-15)
    strat = GpuStrategy(Database(cols.astype(np.int32), [int(a) for a in arities]))
    specs = [QuerySpec(q[0], tuple(q[1:])) for q in queries]
    a = strat.query_batch(specs, loglik=True, mi=True, nnz=True)
    b = strat.query_batch(specs, loglik=True, mi=True, nnz=True, tables=True)
    assert np.array_equal(a["nnz"], onnz) and np.array_equal(b["nnz"], onnz)
    assert all(rel_close(x, y, 1e-12) for x, y in zip(a["loglik"], b["loglik"]))
    assert all(rel_close(x, y, 1e-9) for x, y in zip(a["loglik"], oll))
    otabs = O.dense_tables(cols, arities, queries)[0]
    assert np.array_equal(b["tables"], otabs)
