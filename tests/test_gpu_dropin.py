"""The per-query drop-in path: GpuStrategy.query -> cs_query_one (K8 latency class, one launch,
results in mapped host memory) and its fall-back to the batch path for queries outside the
class.  Reference: Strategy.query (harness.py:44-90), timed per call by bench_random
(harness.py:222-275)."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from conftest import rel_close

pytestmark = pytest.mark.gpu

import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200._native import CS_WANT_TABLES  # noqa: E402
from paper_1804_04640_b200.engine import GpuDatabase  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return cs.shared_context(0)


@pytest.mark.parametrize("m", [1, 3, 4, 5, 1000, 4097, 262_144])
def test_query_one_vs_oracle(ctx, m):
    rng = np.random.default_rng(m)
    ar = [2, 3, 4, 5, 7, 2, 3, 16, 2, 3, 255]
    data = np.vstack([rng.integers(0, a, m) for a in ar]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, ar)
    qs = [(0,), (1, 0), (3, 2, 1), (7, 4, 3), (10, 0), (2, 0, 1, 3, 5, 6, 8, 9), (4, 3, 7, 1)]
    _, _, oll, omi, onnz = O.dense_tables(data, ar, qs, want_tables=False)
    otabs, ooff, _, _, _ = O.dense_tables(data, ar, qs)
    for i, q in enumerate(qs):
        v = np.asarray(q, dtype=np.int32)
        ll, mi, nnz = np.zeros(1), np.zeros(1), np.zeros(1, np.int64)
        gdb.query_one(v, 0, loglik=ll, mi=mi, nnz=nnz)
        assert nnz[0] == onnz[i] and rel_close(ll[0], oll[i], 1e-9)
        assert abs(mi[0] - omi[i]) <= 1e-9 * (abs(oll[i]) + 1) / m + 1e-15
        cells = int(np.prod([ar[x] for x in q]))
        tab = np.zeros(cells, np.uint32)
        gdb.query_one(v, CS_WANT_TABLES, tables=tab)
        assert np.array_equal(tab, otabs[ooff[i]:ooff[i] + cells])


def test_query_one_fallbacks_and_device_outputs(ctx, monkeypatch):
    """Queries outside the latency class (> 8 variables, > 49,152 cells, rows above the limit)
    go through cs_query_batch and give the same answers; device output pointers work."""
    import torch

    rng = np.random.default_rng(3)
    n, m = 12, 20_000
    ar = [2] * 9 + [200, 250, 3]
    data = np.vstack([rng.integers(0, a, m) for a in ar]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, ar)
    qs = [tuple(range(9)), (9, 10), (11, 0, 1)]
    _, _, oll, _, onnz = O.dense_tables(data, ar, qs, want_tables=False)
    for limit in ("262144", "100"):
        monkeypatch.setenv("CS_ONE_MAX_ROWS", limit)
        for i, q in enumerate(qs):
            ll, nnz = np.zeros(1), np.zeros(1, np.int64)
            gdb.query_one(np.asarray(q, np.int32), 0, loglik=ll, nnz=nnz)
            assert nnz[0] == onnz[i] and rel_close(ll[0], oll[i], 1e-9)
    monkeypatch.delenv("CS_ONE_MAX_ROWS")
    dll = torch.zeros(1, dtype=torch.float64, device="cuda")
    dtab = torch.zeros(3 * 4, dtype=torch.int32, device="cuda")
    gdb.query_one(np.asarray((11, 0, 1), np.int32), CS_WANT_TABLES, tables=dtab, loglik=dll)
    torch.cuda.synchronize()
    assert rel_close(float(dll.item()), oll[2], 1e-9)
    otab, _, _, _, _ = O.dense_tables(data, ar, [(11, 0, 1)])
    assert np.array_equal(dtab.cpu().numpy().view(np.uint32), otab)


def test_query_one_errors(ctx):
    gdb = GpuDatabase.from_columns(ctx, np.zeros((3, 10), np.uint8), [2, 2, 2])
    with pytest.raises(cs.InvalidQueryError, match="out of range"):
        gdb.query_one(np.asarray([0, 5], np.int32))
    with pytest.raises(cs.InvalidQueryError, match="repeats variable 1"):
        gdb.query_one(np.asarray([1, 1], np.int32))


def test_strategy_query_all_aggregators(reference_cases):
    """GpuStrategy.query with every aggregator kind on a golden case, including the reference's
    own aggregator objects when baseline/_ref is importable (duck-typed protocol)."""
    from conftest import case_db, golden_records

    case = reference_cases["synthetic-mixed-arity"]
    db = case_db(case)
    s = cs.GpuStrategy(db)
    for q in case["queries"]:
        qs = cs.QuerySpec(q["target"], tuple(q["parents"]))
        col = cs.RecordCollector()
        s.query(qs, col)
        assert {(r.config, r.k, r.n_ijk, r.n_ij) for r in col.result()} == golden_records(q)
        ll = cs.LogLikelihood()
        s.query(qs, ll)
        assert rel_close(ll.result(), q["loglik"], 1e-9)
        mdl = cs.MdlScore.for_query(db, qs)
        s.query(qs, mdl)
        assert rel_close(mdl.result(), q["mdl"], 1e-9)
        sink = cs.NullSink()
        s.query(qs, sink)
        assert sink.count == len(golden_records(q))


def test_query_one_cells_record_stream(ctx):
    """cs_query_one_cells: the non-zero cells in cell order with N_ij; CS_ERR_UNSUPPORTED for a
    query outside the single-query class (the strategy then compacts through a plan)."""
    import ctypes

    from paper_1804_04640_b200 import _native as N

    rng = np.random.default_rng(12)
    m = 30_000
    ar = [3, 4, 2, 5, 250, 200]
    data = np.vstack([rng.integers(0, a, m) for a in ar]).astype(np.uint8)
    data[1, data[0] == 2] = 0  # structural zeros
    gdb = GpuDatabase.from_columns(ctx, data, ar)
    for q in [(0,), (1, 0), (3, 1, 0, 2), (2, 3)]:
        cells = int(np.prod([ar[v] for v in q]))
        ci, a, b = (np.zeros(cells, np.int64) for _ in range(3))
        nz = np.zeros(1, np.int64)
        v = np.asarray(q, np.int32)
        N.check(N.lib.cs_query_one_cells(gdb.handle, len(q), v.ctypes.data, ci.ctypes.data, a.ctypes.data,
                                         b.ctypes.data, nz.ctypes.data))
        t, _, _, _, _ = O.dense_tables(data, ar, [q])
        want = np.flatnonzero(t)
        n = int(nz[0])
        assert np.array_equal(ci[:n], want)
        assert np.array_equal(a[:n], t[want])
        r_t = ar[q[0]]
        assert np.array_equal(b[:n], t.reshape(-1, r_t).sum(axis=1)[want // r_t])
    v = np.asarray((4, 5), np.int32)  # 50,000 cells: outside the class
    big = np.zeros(50_000, np.int64)
    nz = np.zeros(1, np.int64)
    rc = N.lib.cs_query_one_cells(gdb.handle, 2, v.ctypes.data, big.ctypes.data, big.ctypes.data,
                                  big.ctypes.data, nz.ctypes.data)
    assert rc == N.CS_ERR_UNSUPPORTED
    s = cs.GpuStrategy(cs.Database(data.astype(np.int32), ar))
    col = cs.RecordCollector()
    s.query(cs.QuerySpec(4, (5,)), col)  # through the plan + K5 path
    assert len(col.result()) == int(np.count_nonzero(O.dense_tables(data, ar, [(4, 5)])[0]))
