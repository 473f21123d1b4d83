"""K7, the bitmap query class (survey 8(f)3; reference bitmap.py:69-128, Alg. 1): binary
queries of <= 4 variables answered from state-1 bit planes (AND + popcount of every variable
subset, then an in-place superset -> cell transform).  Parity against the oracle, forced on
(CS_BITMAP=1) and compared with the histogram classes (CS_BITMAP=0) on the same plans."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

import oracle as O
from conftest import case_db, golden_records, rel_close

pytestmark = pytest.mark.gpu

import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200._native import CS_WANT_TABLES  # noqa: E402
from paper_1804_04640_b200.engine import GpuDatabase, QueryPlan  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return cs.shared_context(0)


def _classes(capfd):
    err = capfd.readouterr().err
    line = [x for x in err.splitlines() if "plan_build: classes" in x][-1]
    return {kv.split("=")[0]: int(kv.split("=")[1]) for kv in line.split("classes ")[1].split()}


def _run(gdb, qs, flags=CS_WANT_TABLES, mi=True):
    plan = QueryPlan(gdb, qs, flags)
    tabs = np.zeros(plan.total_cells, dtype=np.uint32)
    ll = np.zeros(plan.nq)
    miv = np.zeros(plan.nq)
    nnz = np.zeros(plan.nq, dtype=np.int64)
    plan.execute(tables=tabs, loglik=ll, mi=miv if mi else None, nnz=nnz)
    plan.close()
    return tabs, ll, miv, nnz


@pytest.mark.parametrize("m", [1, 31, 32, 33, 1000, 32768, 32768 * 17 + 5, 1_000_003])
def test_bitmap_class_vs_oracle_ragged(ctx, monkeypatch, capfd, m):
    rng = np.random.default_rng(m)
    n = 7
    p = rng.uniform(0.05, 0.95, n)
    data = (rng.random((n, m)) < p[:, None]).astype(np.uint8)
    data[3] = 1  # a constant variable
    gdb = GpuDatabase.from_columns(ctx, data, [2] * n)
    gdb.bitmap_build()
    qs = [q for k in (1, 2, 3, 4) for q in itertools.islice(itertools.permutations(range(n), k), 0, None, 7)]
    monkeypatch.setenv("CS_BITMAP", "1")
    monkeypatch.setenv("CS_TRACE", "1")
    tabs, ll, mi, nnz = _run(gdb, qs)
    assert _classes(capfd)["bitmap"] == len(qs)
    monkeypatch.setenv("CS_BITMAP", "0")
    tabs0, ll0, mi0, nnz0 = _run(gdb, qs)
    assert _classes(capfd)["bitmap"] == 0
    otabs, _, oll, omi, onnz = O.dense_tables(data, [2] * n, qs)
    assert np.array_equal(tabs, otabs) and np.array_equal(tabs0, otabs)
    assert np.array_equal(nnz, onnz)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(ll, oll))
    assert np.allclose(mi, omi, rtol=1e-9, atol=1e-12)


def test_bitmap_class_mixed_batch_and_records(ctx, monkeypatch, capfd, reference_cases):
    """Bitmap-class queries next to histogram-class ones in one plan (mixed arities), and the
    drop-in strategy's record stream on the reference's binary golden cases."""
    for name in ("synthetic-binary", "synthetic-wide-binary"):
        case = reference_cases[name]
        db = case_db(case)
        monkeypatch.setenv("CS_BITMAP", "1")
        s = cs.GpuStrategy(db)  # builds the bit planes
        for q in case["queries"]:
            col = cs.RecordCollector()
            s.query(cs.QuerySpec(q["target"], tuple(q["parents"])), col)
            got = {(r.config, r.k, r.n_ijk, r.n_ij) for r in col.result()}
            if len(q["parents"]) <= 3:
                assert got == golden_records(q)
    rng = np.random.default_rng(5)
    n, m = 10, 200_000
    ar = [2, 2, 2, 2, 2, 3, 4, 2, 5, 2]  # 5-ary variable: no 2-bit column copy
    data = np.vstack([rng.integers(0, a, m) for a in ar]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, ar)
    gdb.bitmap_build()
    qs = [tuple(int(x) for x in rng.choice(n, int(rng.integers(1, 6)), replace=False)) for _ in range(300)]
    monkeypatch.setenv("CS_BITMAP", "-1")
    monkeypatch.setenv("CS_TRACE", "1")
    tabs, ll, mi, nnz = _run(gdb, qs)
    cls = _classes(capfd)
    assert 0 < cls["bitmap"] < len(qs)
    otabs, _, oll, omi, onnz = O.dense_tables(data, ar, qs)
    assert np.array_equal(tabs, otabs) and np.array_equal(nnz, onnz)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(ll, oll))


def test_bitmap_class_one_shot_and_partial(ctx, monkeypatch):
    """The one-shot chunked cs_query_batch and the instance-shard flag (CS_PARTIAL tables,
    cs_plan_score after the merge) on bitmap-class queries."""
    from paper_1804_04640_b200._native import CS_PARTIAL
    from paper_1804_04640_b200.engine import encode_queries

    monkeypatch.setenv("CS_BITMAP", "1")
    rng = np.random.default_rng(8)
    n, m = 6, 100_001
    data = (rng.random((n, m)) < 0.3).astype(np.uint8)
    qs = [tuple(int(x) for x in rng.choice(n, int(rng.integers(1, 5)), replace=False)) for _ in range(5000)]
    otabs, _, oll, _, _ = O.dense_tables(data, [2] * n, qs)
    gdb = GpuDatabase.from_columns(ctx, data, [2] * n)
    gdb.bitmap_build()
    off, flat = encode_queries(qs)
    tabs = np.zeros(len(otabs), dtype=np.uint32)
    ll = np.zeros(len(qs))
    gdb.query_batch(off, flat, CS_WANT_TABLES, tables=tabs, loglik=ll)
    assert np.array_equal(tabs, otabs)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(ll, oll))
    # two row shards, partial tables summed on the host, then scored with the global m
    half = m // 2
    parts = []
    for r0, r1 in ((0, half), (half, m)):
        g = GpuDatabase.from_columns(ctx, np.ascontiguousarray(data[:, r0:r1]), [2] * n)
        g.bitmap_build()
        g.set_total_rows(m)
        plan = QueryPlan(g, qs[:500], CS_WANT_TABLES | CS_PARTIAL)
        t = np.zeros(plan.total_cells, dtype=np.uint32)
        plan.execute(tables=t)
        parts.append((plan, t))
    merged = parts[0][1] + parts[1][1]
    assert np.array_equal(merged, otabs[: len(merged)])
    ll2 = np.zeros(500)
    parts[0][0].score(merged, loglik=ll2)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(ll2, oll[:500]))
