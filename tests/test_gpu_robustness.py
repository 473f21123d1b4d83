"""Robustness of the C ABI at the edges VERDICT r1 found (What's weak 7, 8, 12):

* batches past the 65,535 grid.y limit (count_batch of 200,000 itemsets, mine_rules levels
  of tens of thousands of candidates, > 65,535-query generic / many-variable lists);
* one shared context driven from many threads by two strategies over two databases
  (reference harness.py:258-267 runs bench_random's queries from a thread pool);
* the opt-in 16-bit counter path (CS_HALF) at its replica bound;
* chunked one-shot batches: global query index in errors, no partial outputs;
* row counts beyond the uint32 tables.
"""

from __future__ import annotations

import itertools
import threading

import numpy as np
import pytest

import oracle as O
from conftest import rel_close

pytestmark = pytest.mark.gpu

import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200._native import CS_WANT_TABLES  # noqa: E402
from paper_1804_04640_b200.database import Database, UnsupportedQueryError  # noqa: E402
from paper_1804_04640_b200.engine import GpuDatabase, QueryPlan  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return cs.shared_context(0)


def _binary_db(n, m, seed, dens=(0.05, 0.6)):
    rng = np.random.default_rng(seed)
    p = rng.uniform(*dens, n)
    data = (rng.random((n, m)) < p[:, None]).astype(np.int32)
    return Database(data, [2] * n)


@pytest.mark.parametrize("bitmaps", [True, False], ids=["bitmap", "scan"])
def test_count_batch_200k_itemsets(bitmaps):
    db = _binary_db(200, 5000, 11)
    s = cs.GpuStrategy(db, bitmaps=bitmaps)
    rng = np.random.default_rng(3)
    asg = []
    for i in range(200_000):
        k = 1 + i % 4
        vs = tuple(sorted(int(x) for x in rng.choice(200, k, replace=False)))
        asg.append(cs.Assignment(vs, tuple(int(x) for x in rng.integers(0, 2, k))))
    got = s.count_batch(asg)
    u8 = db.columns_u8()
    planes = {(v, st): O.bitmap_planes(u8[v], st) for v in range(200) for st in (0, 1)}
    want = O.bitmap_counts(planes, [tuple(zip(a.variables, a.states)) for a in asg], db.m)
    assert np.array_equal(got, want)


def test_mine_rules_wide_levels():
    """200 binary items, low support: level 2 has 19,110 candidates and level 3 504,024 (one
    count_batch each, far past grid.y's 65,535); rules equal those mined with oracle counts."""
    db = _binary_db(200, 3000, 5, dens=(0.05, 0.5))
    s = cs.GpuStrategy(db)
    u8 = db.columns_u8()
    planes = {v: O.bitmap_planes(u8[v], 1) for v in range(db.n)}

    class OracleCounts:  # the reference's count(a) semantics, bitmap_count restated
        def count(self, a):
            return int(O.bitmap_counts({(v, 1): planes[v] for v in a.variables},
                                       [tuple((v, 1) for v in a.variables)], db.m, nthreads=1)[0])

        def count_batch(self, al):
            al = list(al)
            return O.bitmap_counts({(v, 1): planes[v] for v in range(db.n)},
                                   [tuple((v, 1) for v in a.variables) for a in al], db.m)

    got = cs.mine_rules(db, s, min_support=0.05, min_confidence=0.3, max_size=3)
    want = cs.mine_rules(db, OracleCounts(), min_support=0.05, min_confidence=0.3, max_size=3)
    assert len(got) > 1000 and got == want


def test_generic_class_over_65535_queries(ctx):
    """> 8 variables per query (K1g) for 70,000 queries in one plan."""
    rng = np.random.default_rng(9)
    n, m = 12, 700
    data = rng.integers(0, 2, (n, m)).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, [2] * n)
    qs = [tuple(int(x) for x in rng.permutation(n)[:9]) for _ in range(70_000)]
    plan = QueryPlan(gdb, qs)
    ll = np.zeros(plan.nq)
    nnz = np.zeros(plan.nq, dtype=np.int64)
    plan.execute(loglik=ll, nnz=nnz)
    _, _, oll, _, onnz = O.dense_tables(data, [2] * n, qs[:3000], want_tables=False)
    assert np.array_equal(nnz[:3000], onnz)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(ll[:3000], oll))
    _, _, oll2, _, onnz2 = O.dense_tables(data, [2] * n, qs[-3000:], want_tables=False)
    assert np.array_equal(nnz[-3000:], onnz2)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(ll[-3000:], oll2))


def test_shared_context_two_databases_threads():
    """Two strategies over two databases share one context; 8 threads hammer both (fused LL,
    record streams, one-shot batches, point counts); every answer matches the oracle."""
    dbs = [cs.generate_synthetic(9, 20_000, [2, 3, 4, 5, 2, 3, 4, 5, 3], seed=s) for s in (1, 2)]
    strats = [cs.GpuStrategy(d) for d in dbs]
    rng = np.random.default_rng(4)
    jobs = []
    for i in range(400):
        which = i % 2
        vs = [int(x) for x in rng.choice(9, 1 + i % 4, replace=False)]
        jobs.append((which, cs.QuerySpec(vs[0], tuple(vs[1:]))))
    want = {}
    for which in (0, 1):
        qs = [(q.target, *q.parents) for w_, q in jobs if w_ == which]
        _, _, ll, _, nnz = O.dense_tables(dbs[which].columns_u8(), dbs[which].arities, qs, want_tables=False)
        for q, a, b in zip([q for w_, q in jobs if w_ == which], ll, nnz):
            want[(which, q)] = (a, int(b))
    errors = []

    def worker(t):
        try:
            for j, (which, q) in enumerate(jobs[t::8]):
                s = strats[which]
                mode = (t + j) % 3
                if mode == 0:
                    agg = cs.LogLikelihood()
                    s.query(q, agg)
                    assert rel_close(agg.result(), want[(which, q)][0], 1e-9)
                elif mode == 1:
                    sink = cs.NullSink()
                    s.query(q, sink)
                    assert sink.count == want[(which, q)][1]
                else:
                    out = s.query_batch([q, q], loglik=True, nnz=True)
                    assert out["nnz"].tolist() == [want[(which, q)][1]] * 2
                a = cs.Assignment((q.target,), (0,))
                assert s.count(a) == int((dbs[which].columns_u8()[q.target] == 0).sum())
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    th = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errors, errors[:3]


def test_bench_random_parallel_threads():
    """bench_random(parallel=8) (harness.py:235-275) on the shared context: record counts are
    the oracle's non-zero cell counts."""
    db = cs.generate_synthetic(10, 5000, [2, 3, 4, 2, 3, 4, 2, 3, 4, 5], seed=8)
    res = cs.bench_random(db, num_queries=60, seed=3, repetitions=2, parallel=8)
    qs = [(q.target, *q.parents) for q in res.stream.queries]
    _, _, _, _, nnz = O.dense_tables(db.columns_u8(), db.arities, qs, want_tables=False)
    got = {t.query_id: t.record_count for t in res.timings}
    assert [got[i] for i in range(len(qs))] == nnz.tolist()


@pytest.mark.parametrize("m", [65535 * 32, 1_900_000], ids=["old_bound", "half_enabled"])
def test_half_counters_at_replica_bound(ctx, monkeypatch, m):
    """CS_HALF on a near-constant column whose one segment sits at (or below) the old bound
    (65535 * 32 rows): no 16-bit counter may wrap into its neighbour."""
    monkeypatch.setenv("CS_HALF", "1")
    monkeypatch.setenv("CS_NIBBLE", "0")  # uint8 layout: 16 rows per vector (the worst case)
    n = 5
    data = np.zeros((n, m), dtype=np.uint8)
    data[:, ::7] = 3  # mostly one cell, a second one every 7th row
    gdb = GpuDatabase.from_columns(ctx, data, [5] * n)
    qs = [tuple(range(n))] * 600  # enough queries for one segment per query
    plan = QueryPlan(gdb, qs, CS_WANT_TABLES)
    tabs = np.zeros(plan.total_cells, dtype=np.uint32)
    plan.execute(tables=tabs)
    ot, _, _, _, _ = O.dense_tables(data, [5] * n, qs[:1])
    for i in (0, 299, 599):
        assert np.array_equal(tabs[plan.table_off[i]:plan.table_off[i] + plan.cells[i]], ot)


def test_chunked_batch_errors_name_global_index(ctx, monkeypatch):
    monkeypatch.setenv("CS_QB_CHUNKS", "3")
    rng = np.random.default_rng(1)
    data = rng.integers(0, 3, (6, 500)).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, [3] * 6)
    qs = [(i % 6, (i + 1) % 6) for i in range(5000)]
    qs[4321] = (2, 4, 2)  # repeats a variable, in the last chunk
    from paper_1804_04640_b200.engine import encode_queries

    off, flat = encode_queries(qs)
    ll = np.full(len(qs), 7.0)
    with pytest.raises(cs.InvalidQueryError, match="query 4321 repeats variable 2"):
        gdb.query_batch(off, flat, 0, loglik=ll)
    assert (ll == 7.0).all()  # validated before the first chunk ran: nothing written


def test_row_count_limit(ctx):
    with pytest.raises(UnsupportedQueryError, match="2\\^32"):
        GpuDatabase.empty(ctx, 1, 2**32, [2])
    g = GpuDatabase.from_columns(ctx, np.zeros((1, 10), np.uint8), [2])
    with pytest.raises(UnsupportedQueryError):
        g.set_total_rows(2**32)
