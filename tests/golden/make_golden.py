#!/usr/bin/env python3
"""Regenerate the golden fixtures of tests/golden/ from the reference implementation itself.

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden.py

It imports the UNMODIFIED reference package read-only from
/root/reference/pkg/src (countstream) and records its outputs:

* reference_cases.json -- the six cases of the reference's own binding golden
  files (pkg/bindings/test/golden/generate.py CASES: same sources and queries),
  recomputed through the reference API: records (oracle_query), loglik
  (radix_query + LogLikelihood), mdl (mdl_score via radix), learn_parents,
  mine_rules.  The script asserts they equal the committed upstream JSONs,
  which pins this run of the reference to the upstream capture;
* random_sweep.json.gz -- seeded random databases in the reference's correctness
  regime (conftest.make_random_db: n<=10, m<=512, arity<=5) with queries, their
  record sets (oracle_query), LL / MDL (radix) and point counts (oracle_count);
* cfg1.npz            -- BASELINE configs[0] in full: the database built by the
  reference generator (cli._parse_synthetic) and, for all 1,000 queries, dense
  N_ijk tables (from radix_query record streams) and LL (radix + LogLikelihood).
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

import numpy as np  # noqa: E402

import countstream as cs  # noqa: E402  (the reference)
from countstream.cli import _parse_synthetic  # noqa: E402
from countstream.harness import RadixStrategy  # noqa: E402

FIXTURE_CSV = REF / "tests" / "data" / "fixture.csv"

# the reference's binding golden cases (pkg/bindings/test/golden/generate.py CASES)
CASES = {
    "fixture": ({"csv": "fixture"}, [(1, [0, 2]), (0, []), (2, [0, 1])], 2, None),
    "synthetic-ternary": ({"n": 4, "m": 120, "arity": 3, "seed": 11}, [(0, [1, 2]), (3, [0])], 2, None),
    "synthetic-binary": ({"n": 6, "m": 400, "arity": 2, "seed": 22}, [(5, [0, 3]), (2, [1, 4, 5])], 2,
                         (0.2, 0.3, 6)),
    "synthetic-mixed-arity": ({"n": 8, "m": 1000, "arity": [2, 4], "seed": 33},
                              [(2, [4, 6, 7]), (0, [1, 2, 3])], 2, None),
    "synthetic-quaternary": ({"n": 5, "m": 64, "arity": 4, "seed": 44}, [(4, [0, 1]), (1, [2, 3])], 3, None),
    "synthetic-wide-binary": ({"n": 7, "m": 2048, "arity": 2, "seed": 55}, [(3, [1, 2])], 2, (0.15, 0.5, 4)),
}


def spec_of(src) -> str:
    a = src["arity"]
    part = f"{a[0]}-{a[1]}" if isinstance(a, list) else str(a)
    return f"n={src['n']},m={src['m']},arity={part},seed={src['seed']}"


def load_source(src):
    if src.get("csv") == "fixture":
        return cs.load_csv(FIXTURE_CSV, delimiter=",")
    return _parse_synthetic(spec_of(src), 0)


def recs_json(records):
    rs = sorted(records, key=lambda r: (r.config, r.k))
    return [{"config": [list(c) for c in r.config], "k": r.k, "n_ijk": r.n_ijk, "n_ij": r.n_ij} for r in rs]


def run_query(db, strat, t, ps):
    q = cs.QuerySpec(t, tuple(ps))
    recs = cs.oracle_query(db, q)
    agg = cs.LogLikelihood()
    strat.query(q, agg)
    return {"target": t, "parents": list(ps), "records": recs_json(recs), "loglik": agg.result(),
            "mdl": cs.mdl_score(db, q, strat)}


def reference_cases():
    out = {}
    for name, (src, queries, learn, rules) in CASES.items():
        db = load_source(src)
        built, _ = cs.make_strategies(db, ("radix", "bitmap"))
        case = {"source": src, "n": db.n, "m": db.m, "arities": db.arities.tolist(),
                "queries": [run_query(db, built["radix"], t, ps) for t, ps in queries]}
        if src.get("csv") == "fixture":
            case["data"] = db.data.tolist()
        res = cs.learn_parents(db, built["radix"], max_parents=learn)
        case["learn"] = {"maxParents": learn,
                         "parentSets": [{"target": r.target, "parents": list(r.parents), "score": r.score}
                                        for r in res]}
        if rules:
            s, c, k = rules
            rr = cs.mine_rules(db, built["bitmap"], s, c, k)
            case["rules"] = {"minSupport": s, "minConfidence": c, "maxSize": k,
                             "rules": sorted(({"antecedent": list(r.antecedent), "consequent": r.consequent,
                                               "support": r.support, "confidence": r.confidence} for r in rr),
                                             key=lambda r: (r["antecedent"], r["consequent"]))}
        # pin against the reference's committed golden capture
        up = json.loads((REF / "bindings" / "test" / "golden" / f"{name}.json").read_text())
        for mine, theirs in zip(case["queries"], up["queries"]):
            assert mine["records"] == theirs["records"], name
            assert abs(mine["loglik"] - theirs["loglik"]) <= 1e-12 * max(1, abs(theirs["loglik"])), name
            assert abs(mine["mdl"] - theirs["mdl"]) <= 1e-12 * max(1, abs(theirs["mdl"])), name
        assert [p["parents"] for p in case["learn"]["parentSets"]] == \
            [p["parents"] for p in up["learn"]["parentSets"]], name
        if rules:
            assert [(r["antecedent"], r["consequent"]) for r in case["rules"]["rules"]] == \
                [(r["antecedent"], r["consequent"]) for r in up["rules"]["rules"]], name
        out[name] = case
    return out


def random_sweep(seed=20241020, ndb=60, nq=5, npoint=6):
    rng = np.random.default_rng(seed)
    dbs = []
    for _ in range(ndb):
        n = int(rng.integers(2, 11))
        m = int(rng.integers(1, 513))
        ar = rng.integers(2, 6, size=n).tolist()
        s = int(rng.integers(0, 2**31))
        db = cs.generate_synthetic(n, m, ar, seed=s)
        radix = RadixStrategy(db)
        qs = []
        for _ in range(nq):
            t = int(rng.integers(0, n))
            size = int(rng.integers(0, n))
            others = [v for v in range(n) if v != t]
            ps = [int(p) for p in rng.choice(others, size=min(size, len(others)), replace=False)] if size else []
            qs.append(run_query(db, radix, t, ps))
        pts = []
        for _ in range(npoint):
            size = int(rng.integers(0, n + 1))
            vs = sorted(int(v) for v in rng.choice(n, size=size, replace=False))
            ss = [int(rng.integers(0, ar[v])) for v in vs]
            pts.append({"vars": vs, "states": ss, "count": cs.oracle_count(db, cs.Assignment(vs, ss))})
        dbs.append({"n": n, "m": m, "arities": ar, "seed": s, "queries": qs, "points": pts})
    return {"seed": seed, "dbs": dbs}


def cfg1_golden(seed=1):
    from paper_1804_04640_b200 import workloads

    w = workloads.cfg1(seed)
    ref_db = _parse_synthetic(f"n=20,m=10000,arity=2-4,seed={seed}", 0)
    assert np.array_equal(ref_db.data, w.host_db.data), "cfg1 restated generator differs from reference"
    radix = RadixStrategy(ref_db)
    ar = ref_db.arities
    tables, offs, lls = [], [0], []
    for (t, *ps) in w.queries:
        q = cs.QuerySpec(t, tuple(ps))
        col = cs.RecordCollector()
        radix.query(q, col)
        strides = {}
        s = int(ar[t])
        for p in ps:
            strides[p] = s
            s *= int(ar[p])
        tab = np.zeros(s, dtype=np.uint32)
        for r in col.result():
            tab[r.k + sum(st * strides[v] for v, st in r.config)] = r.n_ijk
        tables.append(tab)
        offs.append(offs[-1] + s)
        agg = cs.LogLikelihood()
        radix.query(q, agg)
        lls.append(agg.result())
    np.savez_compressed(HERE / "cfg1.npz", queries=np.array(w.queries, dtype=np.int32),
                        tables=np.concatenate(tables), table_off=np.array(offs[:-1], dtype=np.int64),
                        loglik=np.array(lls), data=ref_db.data.astype(np.uint8),
                        arities=np.asarray(ar, dtype=np.int32), seed=np.array(seed))


def main():
    (HERE / "reference_cases.json").write_text(json.dumps(reference_cases(), indent=0) + "\n")
    with gzip.open(HERE / "random_sweep.json.gz", "wt") as fh:
        json.dump(random_sweep(), fh)
    cfg1_golden()
    print("wrote reference_cases.json random_sweep.json.gz cfg1.npz")


if __name__ == "__main__":
    main()
