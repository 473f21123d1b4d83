"""Pin the oracle (CPU restatements in oracle/) to the reference's golden vectors.

Everything the GPU parity tests trust comes from here: the numpy definitional
oracle and the C radix restatement must reproduce, exactly, the record sets,
counts and scores captured from the reference implementation
(tests/golden/make_golden.py) and the reference's hand-derived KATs.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import oracle as O
from conftest import (
    FIXTURE_X1_GIVEN_X0_X2,
    FIXTURE_X2_EMPTY,
    case_db,
    golden_records,
    rel_close,
    sweep_db,
)


def test_fixture_kats_numpy_oracle(reference_cases):
    db = case_db(reference_cases["fixture"])
    assert O.oracle_records(db.data, db.arities, 1, (0, 2)) == FIXTURE_X1_GIVEN_X0_X2
    assert O.oracle_records(db.data, db.arities, 1, (2, 0)) == FIXTURE_X1_GIVEN_X0_X2
    assert O.oracle_records(db.data, db.arities, 1, (0, 2), exhaustive_limit=0) == FIXTURE_X1_GIVEN_X0_X2
    assert O.oracle_records(db.data, db.arities, 2, ()) == FIXTURE_X2_EMPTY
    assert O.oracle_count(db.data, (0, 1, 2), (2, 1, 0)) == 2
    assert O.oracle_count(db.data, (0, 1, 2), (0, 0, 0)) == 1
    assert O.oracle_count(db.data, (0, 2), (0, 1)) == 0
    assert O.oracle_count(db.data, (), ()) == 8
    assert [O.oracle_count(db.data, (0,), (s,)) for s in range(3)] == [2, 3, 3]


def test_fixture_kats_radix_restatement(reference_cases):
    db = case_db(reference_cases["fixture"])
    u8 = db.columns_u8()
    for t, ps, want in [(1, (0, 2), FIXTURE_X1_GIVEN_X0_X2), (1, (2, 0), FIXTURE_X1_GIVEN_X0_X2),
                        (2, (), FIXTURE_X2_EMPTY)]:
        tabs, off, ll, nnz = O.radix_tables(u8, db.arities, [(t, *ps)], nthreads=1)
        assert O.records_from_table(tabs, t, ps, db.arities) == want
        assert nnz[0] == len(want)
        assert rel_close(ll[0], O.loglik_of_records(want), 1e-12)


@pytest.mark.parametrize("name", ["fixture", "synthetic-ternary", "synthetic-binary",
                                  "synthetic-mixed-arity", "synthetic-quaternary", "synthetic-wide-binary"])
def test_reference_cases(reference_cases, name):
    case = reference_cases[name]
    db = case_db(case)
    assert db.arities.tolist() == case["arities"]
    queries = [(q["target"], *q["parents"]) for q in case["queries"]]
    tabs, off, ll, nnz = O.radix_tables(db.columns_u8(), db.arities, queries, nthreads=2)
    for i, q in enumerate(case["queries"]):
        want = golden_records(q)
        assert O.oracle_records(db.data, db.arities, q["target"], q["parents"]) == want
        cells = int(np.prod([db.arities[v] for v in queries[i]]))
        got = O.records_from_table(tabs[off[i]:off[i] + cells], q["target"], q["parents"], db.arities)
        assert got == want
        assert nnz[i] == len(want)
        assert rel_close(ll[i], q["loglik"], 1e-12)
        q_i = int(np.prod([db.arities[p] for p in q["parents"]])) if q["parents"] else 1
        assert rel_close(O.mdl_of(ll[i], db.m, int(db.arities[q["target"]]), q_i), q["mdl"], 1e-12)


def test_random_sweep_records_and_scores(random_sweep):
    checked = 0
    for d in random_sweep["dbs"]:
        db = sweep_db(d)
        queries = [(q["target"], *q["parents"]) for q in d["queries"]]
        tabs, off, ll, nnz = O.radix_tables(db.columns_u8(), db.arities, queries, nthreads=4)
        for i, q in enumerate(d["queries"]):
            want = golden_records(q)
            cells = int(np.prod([db.arities[v] for v in queries[i]]))
            got = O.records_from_table(tabs[off[i]:off[i] + cells], q["target"], q["parents"], db.arities)
            assert got == want
            assert rel_close(ll[i], q["loglik"], 1e-12)
            checked += 1
        for p in d["points"]:
            assert O.oracle_count(db.data, p["vars"], p["states"]) == p["count"]
    assert checked >= 250


def test_random_sweep_bitmap_counts(random_sweep):
    for d in random_sweep["dbs"][:30]:
        db = sweep_db(d)
        u8 = db.columns_u8()
        planes = {(v, s): O.bitmap_planes(u8[v], s) for v in range(db.n) for s in range(int(db.arities[v]))}
        its = [tuple(zip(p["vars"], p["states"])) for p in d["points"]]
        got = O.bitmap_counts(planes, its, db.m, nthreads=2)
        assert got.tolist() == [p["count"] for p in d["points"]]


def test_cfg1_full(cfg1_golden):
    g = cfg1_golden
    queries = [tuple(int(v) for v in q) for q in g["queries"]]
    tabs, off, ll, nnz = O.radix_tables(g["data"], g["arities"], queries)
    assert np.array_equal(off, g["table_off"])
    assert np.array_equal(tabs, g["tables"])
    assert np.allclose(ll, g["loglik"], rtol=1e-12, atol=0)


def test_analytic_loglik():
    # functional copy: L = 0 (reference test_acceptance.py:169-176)
    copy = np.repeat(np.arange(3, dtype=np.uint8), 4)[None, :]
    cols = np.vstack([copy, copy])
    _, _, ll, _ = O.radix_tables(cols, [3, 3], [(1, 0)], nthreads=1)
    assert abs(ll[0]) < 1e-12
    # balanced binary column: L = 8 ln 0.5 (:178-184)
    _, _, ll, _ = O.radix_tables(np.array([[0, 0, 0, 0, 1, 1, 1, 1]], dtype=np.uint8), [2], [(0,)])
    assert abs(ll[0] - 8 * math.log(0.5)) < 1e-12


def test_mi_definition():
    rng = np.random.default_rng(7)
    x = rng.integers(0, 3, 400).astype(np.uint8)
    y = ((x + rng.integers(0, 2, 400)) % 3).astype(np.uint8)
    cols = np.vstack([x, y])
    recs = O.oracle_records(cols, [3, 3], 1, (0,))
    mi = O.mi_of_records(recs, 400)
    ll1 = O.loglik_of_records(recs)
    ll0 = O.loglik_of_records(O.oracle_records(cols, [3, 3], 1, ()))
    assert abs(mi - (ll1 - ll0) / 400) < 1e-12
    assert mi > 0


# ---- the direct-count restatements (count_oracle.c) used by the full-size parity tests ------


def test_dense_tables_reference_cases(reference_cases):
    for name, case in reference_cases.items():
        if "queries" not in case:
            continue
        db = case_db(case)
        queries = [(q["target"], *q["parents"]) for q in case["queries"]]
        tabs, off, ll, mi, nnz = O.dense_tables(db.columns_u8(), db.arities, queries, nthreads=2)
        for i, q in enumerate(case["queries"]):
            want = golden_records(q)
            cells = int(np.prod([db.arities[v] for v in queries[i]]))
            got = O.records_from_table(tabs[off[i]:off[i] + cells], q["target"], q["parents"], db.arities)
            assert got == want, (name, i)
            assert nnz[i] == len(want)
            assert rel_close(ll[i], q["loglik"], 1e-12)
            assert abs(mi[i] - O.mi_of_records(want, db.m)) <= 1e-12 * max(1.0, abs(ll[i]) / db.m)


def test_dense_tables_random_sweep_and_cfg1(random_sweep, cfg1_golden):
    for d in random_sweep["dbs"]:
        db = sweep_db(d)
        queries = [(q["target"], *q["parents"]) for q in d["queries"]]
        tabs, off, ll, mi, nnz = O.dense_tables(db.columns_u8(), db.arities, queries, nthreads=2)
        rt, _, rll, _ = O.radix_tables(db.columns_u8(), db.arities, queries, nthreads=2)
        assert np.array_equal(tabs, rt)
        for i, q in enumerate(d["queries"]):
            assert rel_close(ll[i], q["loglik"], 1e-12)
    g = cfg1_golden
    queries = [tuple(int(v) for v in q) for q in g["queries"]]
    tabs, off, ll, _, _ = O.dense_tables(g["data"], g["arities"], queries)
    assert np.array_equal(off, g["table_off"]) and np.array_equal(tabs, g["tables"])
    assert np.allclose(ll, g["loglik"], rtol=1e-12, atol=0)
    # without tables (internal scratch), and over a row prefix of a wider array
    _, _, ll2, _, _ = O.dense_tables(g["data"], g["arities"], queries, want_tables=False)
    assert np.array_equal(ll, ll2)
    wide = np.hstack([g["data"], np.zeros((g["data"].shape[0], 77), np.uint8)])
    _, _, ll3, _, _ = O.dense_tables(wide, g["arities"], queries, want_tables=False, m=g["data"].shape[1])
    assert np.array_equal(ll, ll3)


@pytest.mark.parametrize("n,m,density", [(3, 50, 0.5), (12, 3000, 0.3), (70, 20000, 0.05)])
def test_itemset_enum_matches_bitmap_count(n, m, density):
    import itertools

    rng = np.random.default_rng(n * 1000 + m)
    p = rng.uniform(0, 2 * density, n)
    p[0] = 1.0  # an always-present item (cfg4's clipped p_1)
    cols = (rng.random((n, m)) < p[:, None]).astype(np.uint8)
    pairs, triples = O.itemset_supports_enum(cols, nthreads=3)
    planes = {(v, 1): O.bitmap_planes(cols[v], 1) for v in range(n)}
    combos2 = list(itertools.combinations(range(n), 2))
    want2 = O.bitmap_counts(planes, [tuple((v, 1) for v in c) for c in combos2], m)
    assert [int(pairs[a, b]) for a, b in combos2] == want2.tolist()
    combos3 = list(itertools.combinations(range(n), 3))
    want3 = O.bitmap_counts(planes, [tuple((v, 1) for v in c) for c in combos3], m)
    assert triples.tolist() == want3.tolist()
    for c in combos3[:: max(1, len(combos3) // 50)]:
        assert O.oracle_count(cols, c, (1, 1, 1)) == triples[combos3.index(c)]
