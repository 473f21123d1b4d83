"""Host-side API (CPU): descriptors, loaders, aggregators, drivers' pure logic.

Mirrors the reference's unit tests for the layers this package re-implements on the host
(pkg/tests/test_database.py, test_aggregators.py, test_harness.py) -- same inputs, same
expected values and errors -- plus the workload generators' shapes.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import FIXTURE_ROWS_1BASED, rel_close

import paper_1804_04640_b200 as cs
from paper_1804_04640_b200 import harness, workloads
from paper_1804_04640_b200.database import parse_synthetic


@pytest.fixture
def fixture_csv(tmp_path):
    p = tmp_path / "fixture.csv"
    p.write_text("\n".join(",".join(str(x) for x in r) for r in FIXTURE_ROWS_1BASED) + "\n")
    return p


def test_fixture_shape_and_shift(fixture_csv, reference_cases):
    db = cs.load_csv(fixture_csv, delimiter=",")
    assert (db.n, db.m) == (3, 8)
    assert db.arities.tolist() == [3, 2, 2]
    assert db.data.tolist() == reference_cases["fixture"]["data"]
    assert db.column(0).tolist() == [0, 0, 1, 1, 2, 2, 2, 1]


def test_loader_errors(tmp_path):
    p = tmp_path / "r.csv"
    p.write_text("0,1\n1\n")
    with pytest.raises(cs.DatabaseLoadError, match="row 2"):
        cs.load_csv(p)
    p.write_text("0,1\n1,x\n")
    with pytest.raises(cs.DatabaseLoadError, match="row 2: non-integer"):
        cs.load_csv(p)
    p.write_text("")
    with pytest.raises(cs.DatabaseLoadError, match="no records"):
        cs.load_csv(p)
    p.write_text("0 -1\n")
    with pytest.raises(cs.DatabaseLoadError, match="negative"):
        cs.load_csv(p)
    p.write_text("0 1\n2 0\n")
    db = cs.load_csv(p)  # zero present: kept verbatim, whitespace delimiter
    assert db.data.tolist() == [[0, 2], [1, 0]]
    db = cs.load_csv(p, arities=[5, 4])
    assert db.arities.tolist() == [5, 4]
    with pytest.raises(cs.DatabaseLoadError, match="exceeding declared arity"):
        cs.load_csv(p, arities=[2, 4])
    a = tmp_path / "ar.txt"
    a.write_text("3 4\n")
    assert cs.load_arities(a) == [3, 4]


def test_database_validation_and_immutability():
    with pytest.raises(cs.DatabaseLoadError):
        cs.Database(np.zeros((0, 3), dtype=np.int32))
    with pytest.raises(cs.DatabaseLoadError):
        cs.Database(np.zeros((2, 3), dtype=np.int32), arities=[2])
    db = cs.Database(np.array([[0, 1, 2], [1, 1, 0]]))
    with pytest.raises(ValueError):
        db.data[0, 0] = 5
    rm = db.row_major()
    assert rm.shape == (3, 2) and rm is db.row_major()
    big = cs.Database(np.array([[0, 300]]))
    with pytest.raises(cs.UnsupportedQueryError):
        big.columns_u8()


def test_query_and_assignment_validation():
    with pytest.raises(cs.InvalidQueryError):
        cs.QuerySpec(0, (1, 1))
    with pytest.raises(cs.InvalidQueryError):
        cs.QuerySpec(1, (1,))
    with pytest.raises(cs.InvalidQueryError):
        cs.QuerySpec(-1)
    db = cs.Database(np.zeros((2, 4), dtype=np.int32), arities=[2, 3])
    with pytest.raises(cs.InvalidQueryError):
        cs.QuerySpec(0, (5,)).validate(db)
    with pytest.raises(cs.InvalidQueryError):
        cs.Assignment((0,), (0, 1))
    with pytest.raises(cs.InvalidQueryError):
        cs.Assignment((1,), (3,)).validate(db)
    cs.Assignment((), ()).validate(db)
    assert cs.QuerySpec(1, (0,)).variables == (1, 0)


def test_generator_matches_reference_sample():
    # the reference's frozen PRNG sample (pkg/tests/test_database.py:153-157)
    db = cs.generate_synthetic(3, 4, (2, 3, 4), seed=0)
    assert db.data.tolist() == [[0, 0, 1, 0], [1, 1, 1, 0], [0, 3, 2, 1]]
    a = cs.generate_synthetic(5, 100, 3, seed=7)
    assert np.array_equal(a.data, cs.generate_synthetic(5, 100, 3, seed=7).data)
    assert not np.array_equal(a.data, cs.generate_synthetic(5, 100, 3, seed=8).data)
    db = cs.generate_synthetic(4, 500, (2, 3, 4, 5), seed=3)
    assert db.data.max(axis=1).tolist() == [1, 2, 3, 4]


def test_parse_synthetic_equals_configs0(cfg1_golden):
    db = parse_synthetic("n=20,m=10000,arity=2-4,seed=1")
    assert np.array_equal(db.columns_u8(), cfg1_golden["data"])
    with pytest.raises(ValueError):
        parse_synthetic("n=2,m=3")


def test_aggregators_contract():
    s = cs.NullSink()
    s.accept(1, 2)
    s.accept_block(np.array([1, 1]), np.array([2, 2]))
    assert s.result() == 3
    c = cs.RecordCollector()
    c.accept_record(((0, 1),), 0, 2, 3)
    with pytest.raises(cs.AggregatorContractError):
        c.accept_record(((0, 1),), 0, 2, 3)
    with pytest.raises(cs.AggregatorContractError):
        c.accept(1, 1)
    ll = cs.LogLikelihood()
    ll.accept(2, 4)
    assert rel_close(ll.result(), 2 * math.log(0.5), 1e-15)
    with pytest.raises(cs.AggregatorContractError):
        ll.accept(0, 1)
    with pytest.raises(cs.AggregatorContractError):
        ll.accept_block(np.array([3]), np.array([2]))
    ll2 = cs.LogLikelihood()
    ll2.accept_block(np.array([], dtype=np.int64), np.array([], dtype=np.int64))
    assert ll2.result() == 0.0
    m = cs.MdlScore(8, 2, 3)
    m.accept(4, 8)
    assert rel_close(m.result(), -4 * math.log(0.5) + 0.5 * math.log(8) * 1 * 3, 1e-15)


def test_mutual_information_stream_form():
    mi = cs.MutualInformation(8)
    for cfg, k, n, nij in [(((0, 0),), 0, 4, 4), (((0, 1),), 1, 4, 4)]:
        mi.accept_record(cfg, k, n, nij)
    assert rel_close(mi.result(), math.log(2), 1e-15)


def test_make_strategies_names():
    db = cs.Database(np.zeros((2, 4), dtype=np.int32), arities=[2, 2])
    with pytest.raises(ValueError, match="CPU engine of the reference"):
        cs.make_strategies(db, ("radix",))
    with pytest.raises(ValueError):
        cs.make_strategies(db, ("nope",))
    assert cs.STRATEGY_NAMES == ("gpu",)


def test_random_query_stream_deterministic():
    a = cs.RandomQueryStream.generate(6, 50, 3)
    b = cs.RandomQueryStream.generate(6, 50, 3)
    assert a.queries == b.queries
    assert all(q.target not in q.parents and 1 <= len(q.parents) <= 5 for q in a.queries)
    with pytest.raises(ValueError):
        cs.RandomQueryStream.generate(1, 5, 0)


def test_argmin_tie_rule():
    combos = [(), (1,), (0,), (0, 1)]
    # (0,) and (1,) tie within eps: the lexicographically smaller (0,) wins
    best, bset = harness._argmin_mdl(combos, [10.0, 5.0, 5.0 + 1e-12, 7.0], 1e-9)
    assert bset == (0,) and best == 5.0


class _OracleStrategy(cs.Strategy):
    """CPU stand-in for the batched GPU strategy (tests the drivers' host logic only)."""

    name = "oracle"

    def __init__(self, db):
        import oracle as O

        self.O, self.db = O, db

    def family_scores(self, families):
        qs = [(t, *ps) for t, ps in families]
        _, _, ll, _ = self.O.radix_tables(self.db.columns_u8(), self.db.arities, qs, want_tables=False)
        pen = np.array([0.5 * math.log(self.db.m) * (int(self.db.arities[t]) - 1)
                        * int(np.prod([int(self.db.arities[p]) for p in ps])) for t, ps in families])
        return ll, -ll + pen

    def count_batch(self, assignments):
        return np.array([self.O.oracle_count(self.db.data, a.variables, a.states) for a in assignments])

    def count(self, a):
        return int(self.count_batch([a])[0])


@pytest.mark.parametrize("name", ["fixture", "synthetic-binary", "synthetic-quaternary", "synthetic-wide-binary"])
def test_drivers_reproduce_reference_learn_and_rules(reference_cases, name):
    from conftest import case_db

    case = reference_cases[name]
    db = case_db(case)
    s = _OracleStrategy(db)
    res = cs.learn_parents(db, s, max_parents=case["learn"]["maxParents"])
    assert [list(r.parents) for r in res] == [p["parents"] for p in case["learn"]["parentSets"]]
    for r, p in zip(res, case["learn"]["parentSets"]):
        assert rel_close(r.score, p["score"], 1e-9)
    if "rules" in case:
        rr = case["rules"]
        got = cs.mine_rules(db, s, rr["minSupport"], rr["minConfidence"], rr["maxSize"])
        assert sorted((list(r.antecedent), r.consequent) for r in got) == \
            [(r["antecedent"], r["consequent"]) for r in rr["rules"]]


def test_workload_shapes():
    w3 = workloads.cfg3()
    assert len(w3.queries) == 288_859
    assert all(len(ps) <= 4 and all(p < i for p in ps) for i, ps in enumerate(w3.gen_parents))
    w5 = workloads.cfg5(nq=500)
    assert all(2 <= len(q) <= 8 for q in w5.queries)
    assert all(int(np.prod([int(w5.arities[v]) for v in q])) <= 1 << 24 for q in w5.queries)
    p, c = workloads.zipf_probs()
    assert abs(p.mean() - 0.01) < 1e-9 and p[0] == 1.0
    assert len(workloads.itemsets_of(range(200))) == 1_333_300
    t = workloads.uniform_thresholds(3)
    assert t.tolist() == [1431655766, 2863311531]
