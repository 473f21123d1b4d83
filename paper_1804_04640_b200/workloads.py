"""The five BASELINE.json configurations as seeded synthetic workloads.

The reference measures on public benchmark networks / datasets that are not in
this environment; every config here is seeded synthetic data with the shapes,
sizes and value distributions BASELINE.json states.

* configs[0] (cfg1) is built exactly with the reference's own generator
  (``parse_synthetic("n=20,m=10000,arity=2-4,seed=S")``, cli.py:45-72).
* cfg2..cfg5 are generated on the device by the counter-based generator of
  ``cs_db_generate`` (state = number of per-configuration thresholds the
  32-bit hash of (seed, variable, global row) reaches), so 10-100 GB databases
  never touch the host; ``oracle/gen_twin.py`` recomputes any column in numpy.

Each builder returns a :class:`Workload`: database schema (arities and, per
variable, generator parents + thresholds) plus the query set.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np

from .database import Database, parse_synthetic

__all__ = [
    "Workload",
    "uniform_thresholds",
    "marginal_thresholds",
    "cfg1",
    "cfg2",
    "cfg3",
    "cfg4",
    "cfg5",
    "CONFIGS",
]

TWO32 = float(2**32)


def _rng(seed: int, *spawn) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=spawn)))


def uniform_thresholds(r: int) -> np.ndarray:
    """u >= ceil(s 2^32 / r) for s = 1..r-1 -> state uniform on [0, r)."""
    return np.array([math.ceil(s * TWO32 / r) for s in range(1, r)], dtype=np.uint64).astype(np.uint32)


def marginal_thresholds(p: np.ndarray) -> np.ndarray:
    """Categorical p -> r-1 ascending uint32 thresholds (state s has mass ~p[s])."""
    c = np.cumsum(np.asarray(p, dtype=np.float64))[:-1]
    t = np.clip(np.round(c * TWO32), 0, TWO32 - 1).astype(np.uint64)
    return np.maximum.accumulate(t).astype(np.uint32)


@dataclass
class Workload:
    name: str
    n: int
    m: int
    arities: np.ndarray
    seed: int
    queries: list = field(default_factory=list)          # variable tuples, target first
    gen_parents: list = field(default_factory=list)      # per variable: tuple of parents
    gen_thresholds: list = field(default_factory=list)   # per variable: uint32 array (q*(r-1))
    host_db: Database | None = None                      # cfg1: built on the host
    itemsets: list = field(default_factory=list)         # cfg4: (vars) tuples in state 1
    meta: dict = field(default_factory=dict)

    @property
    def device_generated(self) -> bool:
        return self.host_db is None

    def build_device(self, ctx, row_offset: int = 0, m_shard: int | None = None):
        """Materialise rows [row_offset, row_offset + m_shard) on the device."""
        from .engine import GpuDatabase

        if self.host_db is not None:
            cols = self.host_db.columns_u8()
            if m_shard is not None:
                cols = np.ascontiguousarray(cols[:, row_offset:row_offset + m_shard])
            return GpuDatabase.from_columns(ctx, cols, self.arities)
        ms = self.m if m_shard is None else int(m_shard)
        gdb = GpuDatabase.empty(ctx, self.n, ms, self.arities)
        for v in range(self.n):  # generator parents always precede their child
            gdb.generate(v, self.seed, self.gen_thresholds[v], self.gen_parents[v], row_offset)
        if ms != self.m:
            gdb.set_total_rows(self.m)
        return gdb


def cfg1(seed: int = 1, nq: int = 1000) -> Workload:
    """configs[0]: n=20, arity U{2,3,4}, m=10,000 (reference generator); 1,000 queries of a
    target plus 2 distinct parents; outputs N_ijk tables + fp64 LL."""
    db = parse_synthetic(f"n=20,m=10000,arity=2-4,seed={seed}")
    g = _rng(seed, 3)
    qs = []
    for _ in range(nq):
        v = g.choice(db.n, size=3, replace=False)
        qs.append((int(v[0]), int(v[1]), int(v[2])))
    return Workload("cfg1", db.n, db.m, np.asarray(db.arities), seed, qs, host_db=db)


def cfg2(seed: int = 2, nq: int = 10_000, m: int = 1_000_000, n: int = 100) -> Workload:
    """configs[1]: n=100, arity U{2..5}, per-variable Dirichlet(1) marginals, m=1e6;
    10,000 queries with variable-set size U{1..6}; joint tables only."""
    g = _rng(seed, 2)
    ar = g.integers(2, 6, size=n)
    thr = [marginal_thresholds(g.dirichlet(np.ones(int(r)))) for r in ar]
    gq = _rng(seed, 4)
    qs = []
    for _ in range(nq):
        k = int(gq.integers(1, 7))
        qs.append(tuple(int(x) for x in gq.choice(n, size=k, replace=False)))
    return Workload("cfg2", n, m, ar.astype(np.int64), seed, qs, [()] * n, thr)


def cfg3(seed: int = 3, m: int = 1_000_000, n: int = 37, max_parents: int = 3,
         max_indegree: int = 4) -> Workload:
    """configs[2]: random DAG (n=37, arity U{2,3,4}, in-degree <= 4, Dirichlet(1) CPT rows),
    m=1e6 forward-sampled instances; every (X_i, Pa) with |Pa| <= 3 in learn_parents order."""
    g = _rng(seed, 5)
    ar = g.integers(2, 5, size=n)
    parents, thr = [], []
    for i in range(n):
        d = int(g.integers(0, min(max_indegree, i) + 1))
        ps = tuple(int(x) for x in sorted(g.choice(i, size=d, replace=False))) if d else ()
        q = int(np.prod([int(ar[p]) for p in ps], dtype=np.int64)) if ps else 1
        rows = [marginal_thresholds(g.dirichlet(np.ones(int(ar[i])))) for _ in range(q)]
        parents.append(ps)
        thr.append(np.concatenate(rows) if rows and len(rows[0]) else np.zeros(0, np.uint32))
    qs = []
    for t in range(n):
        others = [v for v in range(n) if v != t]
        for size in range(max_parents + 1):
            for c in itertools.combinations(others, size):
                qs.append((t, *c))
    return Workload("cfg3", n, m, ar.astype(np.int64), seed, qs, parents, thr,
                    meta={"dag_parents": parents})


def zipf_probs(n_items: int = 1000, s: float = 1.1, density: float = 0.01) -> tuple[np.ndarray, float]:
    """p_i = min(1, c i^-s), c solved (bisection) so mean_i p_i = density; returns (p, c)."""
    w = np.arange(1, n_items + 1, dtype=np.float64) ** (-s)
    lo, hi = 0.0, 1.0 / w[-1]
    for _ in range(200):
        c = 0.5 * (lo + hi)
        if np.minimum(1.0, c * w).mean() < density:
            lo = c
        else:
            hi = c
    c = 0.5 * (lo + hi)
    return np.minimum(1.0, c * w), c


def cfg4(seed: int = 4, m: int = 10_000_000, n_items: int = 1000, top: int = 200) -> Workload:
    """configs[3]: binary m=1e7 x 1000 items, inclusion p_i = min(1, c i^-1.1) with mean 1%;
    supports of all 2- and 3-itemsets of the 200 most frequent items (chosen on the device
    by empirical support, ties by index; see select_top_items)."""
    p, c = zipf_probs(n_items, 1.1, 0.01)
    thr = [np.array([min(2**32 - 1, int(round((1.0 - pi) * TWO32)))], dtype=np.uint32) for pi in p]
    ar = np.full(n_items, 2, dtype=np.int64)
    return Workload("cfg4", n_items, m, ar, seed, [], [()] * n_items, thr,
                    meta={"zipf_c": c, "top": top, "p": p})


def select_top_items(supports: np.ndarray, top: int) -> list:
    """Top-`top` items by empirical support, ties broken by lower index."""
    order = sorted(range(len(supports)), key=lambda i: (-int(supports[i]), i))
    return sorted(order[:top])


def itemsets_of(items, sizes=(2, 3)) -> list:
    out = []
    for k in sizes:
        out.extend(itertools.combinations(items, k))
    return out


def cfg5(seed: int = 5, nq: int = 100_000, m: int = 100_000_000, n: int = 1000,
         cap_log2: int = 24) -> Workload:
    """configs[4]: n=1000, arity U{2..8}, uniform states, m=1e8 (100 GB uint8); 100,000
    queries of 2..8 variables with joint state space <= 2^24; merged across instance
    shards, then LL + MI."""
    g = _rng(seed, 2)
    ar = g.integers(2, 9, size=n)
    thr = [uniform_thresholds(int(r)) for r in ar]
    gq = _rng(seed, 6)
    qs = []
    cap = 1 << cap_log2
    while len(qs) < nq:
        k = int(gq.integers(2, 9))
        v = tuple(int(x) for x in gq.choice(n, size=k, replace=False))
        if int(np.prod([int(ar[x]) for x in v], dtype=np.int64)) <= cap:
            qs.append(v)
    return Workload("cfg5", n, m, ar.astype(np.int64), seed, qs, [()] * n, thr)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
