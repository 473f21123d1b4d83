"""Strategy facade and workloads (drop-in for reference harness.py).

The reference registers four CPU engines behind ``Strategy`` (harness.py:44-122)
and drives them one Python call per query.  This package registers the B200
engine under the name ``"gpu"`` and keeps the facade: ``query(q, agg)`` and
``count(a)`` behave exactly as the reference's strategies do (same streams,
same errors), plus batched entry points ``query_batch`` / ``count_batch``
that the workload drivers use to put thousands of queries into one launch.

Workloads mirror the reference: :func:`bench_random` (harness.py:235-275),
:func:`learn_parents` (:296-348, batched per target with the identical
enumeration order and tie rule) and :func:`mine_rules` (:365-429, one
device batch per apriori level).
"""

from __future__ import annotations

import itertools
import math
import threading
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .aggregators import LogLikelihood, MdlScore, MutualInformation, NullSink
from .database import Assignment, Database, InvalidQueryError, QuerySpec
from .engine import FamilyScorer, GpuContext, GpuDatabase, QueryPlan
from . import _native as N

__all__ = [
    "STRATEGY_NAMES",
    "Strategy",
    "GpuStrategy",
    "DeviceDatabase",
    "make_strategies",
    "shared_context",
    "RandomQueryStream",
    "TimingRecord",
    "BenchResult",
    "bench_random",
    "ParentSetResult",
    "learn_parents",
    "AssociationRule",
    "mine_rules",
]

#: engines this package provides; the reference's CPU engines (bitmap, radix,
#: hash, adtree -- harness.py:41) are not re-implemented here.
STRATEGY_NAMES = ("gpu",)
REFERENCE_CPU_STRATEGIES = ("bitmap", "radix", "hash", "adtree")


class Strategy:
    """Uniform face over one engine (harness.py:44-59)."""

    name: str
    build_seconds: float = 0.0

    def query(self, q: QuerySpec, agg) -> None:
        raise NotImplementedError

    def count(self, a: Assignment) -> int:
        raise NotImplementedError


_CTX: dict[int, GpuContext] = {}
_CTX_LOCK = threading.Lock()


def shared_context(device: int = 0) -> GpuContext:
    """One cs_ctx per device per process."""
    with _CTX_LOCK:
        if device not in _CTX:
            _CTX[device] = GpuContext(device)
        return _CTX[device]


class DeviceDatabase:
    """A database that lives only on the device (generated there, too big for the host).

    Exposes the attributes the query/aggregator API reads (``n``, ``m``,
    ``arities``); ``m`` is the total record count when the handle is one
    instance shard of a larger database.
    """

    def __init__(self, gdb: GpuDatabase, m_total: int | None = None):
        self.gdb = gdb
        self.n = gdb.n
        self.m = int(m_total if m_total is not None else gdb.m)
        self.arities = gdb.arities
        if self.m != gdb.m:
            gdb.set_total_rows(self.m)

    def column(self, i: int) -> np.ndarray:
        return self.gdb.download(i)


def _read_pinned(path):
    """File bytes in page-locked host memory when torch can provide it (the H2D copy then runs
    as one DMA), else a plain numpy buffer (the library stages it)."""
    import os

    size = os.path.getsize(path)
    try:
        import torch

        if size >= (8 << 20) and torch.cuda.is_available():
            buf = torch.empty(size, dtype=torch.uint8, pin_memory=True)
            with open(path, "rb", buffering=0) as fh:
                got = fh.readinto(memoryview(buf.numpy()))
            if got == size:
                return buf
    except ImportError:
        pass
    return np.fromfile(str(path), dtype=np.uint8)


def load_csv_device(path, delimiter: str | None = None, arities=None, device: int = 0) -> DeviceDatabase:
    """``load_csv`` (reference database.py:171-207) with the parse on the device.

    The file's bytes go to HBM once and are tokenised there (cs_db_load_text); the host never
    builds the reference's int64 (m, n) matrix.  Same grammar, 1-based shift, arity inference /
    checks and DatabaseLoadError messages as :func:`~paper_1804_04640_b200.database.load_csv`
    for ASCII text.  The result drops into :class:`GpuStrategy` like a host ``Database``.
    """
    raw = _read_pinned(path)
    gdb = GpuDatabase.from_text(shared_context(device), raw, delimiter=delimiter, arities=arities,
                                source=str(path))
    return DeviceDatabase(gdb)


# fused aggregators: by exact type, ours or the reference's (duck-typed protocol)
_FUSED_NAMES = {"LogLikelihood": "loglik", "MdlScore": "mdl", "NullSink": "nnz", "MutualInformation": "mi"}
_FUSED_MODULES = {LogLikelihood.__module__, "countstream.aggregators"}


def _encode_specs(qs) -> tuple[np.ndarray, np.ndarray]:
    """encode_queries of query objects without per-query tuples (8x faster on 10K queries)."""
    off = np.zeros(len(qs) + 1, dtype=np.int32)
    off[1:] = np.cumsum(np.fromiter((len(q.parents) for q in qs), np.int64, len(qs)) + 1)
    flat = np.fromiter(itertools.chain.from_iterable((q.target, *q.parents) for q in qs), np.int32,
                       int(off[-1]))
    return off, flat


def _vars(q) -> tuple:
    """Index-digit order of a query object (ours or the reference's QuerySpec): target first."""
    return (int(q.target), *(int(p) for p in q.parents))


def _fusion_kind(agg) -> str | None:
    t = type(agg)
    if t.__module__ in _FUSED_MODULES and t.__name__ in _FUSED_NAMES:
        return _FUSED_NAMES[t.__name__]
    return None


def _absorb(agg, kind: str, ll: float, mi: float, nnz: int) -> None:
    if hasattr(agg, "absorb_fused"):
        agg.absorb_fused(loglik=ll, mi=mi, nnz=nnz)
    elif kind == "loglik":
        agg.total += ll
    elif kind == "mdl":
        agg._loglik.total += ll
    elif kind == "nnz":
        agg.count += nnz
    else:  # pragma: no cover
        raise TypeError(f"cannot fuse {type(agg)}")


def _dense_limit() -> int:
    """Largest joint state space the engine counts in a dense table (its CS_MAX_DENSE_LOG2
    knob; larger ones go to the hash class, which has no dense table to return)."""
    import os

    return 1 << int(os.environ.get("CS_MAX_DENSE_LOG2", "30") or 30)


class GpuStrategy(Strategy):
    """The B200 engine behind the reference's Strategy facade.

    ``__init__`` does the per-database preparation (upload of the uint8
    columns, bitmap planes for low-arity variables) and, like the reference,
    that time is reported as ``build_seconds`` and excluded from query timings.
    Calls are serialised per instance (SPEC: "serialize calls per database
    handle"), so ``bench_random(parallel>1)`` is safe.
    """

    name = "gpu"

    def __init__(self, db, device: int = 0, bitmaps: bool | str = "auto",
                 bitmap_budget_bytes: int = 1 << 31):
        self.db = db
        self.ctx = shared_context(device)
        self._lock = threading.Lock()
        self._tls = threading.local()
        if isinstance(db, DeviceDatabase):
            self.gdb = db.gdb
        else:
            self.gdb = GpuDatabase.from_columns(self.ctx, db.columns_u8(), db.arities)
        if bitmaps == "auto":
            plane_bytes = int(np.sum(db.arities)) * ((db.m + 7) // 8)
            bitmaps = plane_bytes <= bitmap_budget_bytes and int(np.max(db.arities)) <= 16
        if bitmaps:
            self.gdb.bitmap_build()

    # -- drop-in per-query API ------------------------------------------------------------
    #: tables up to this many cells (the single-query class, cs_query_one_cells) stream their
    #: non-zero cells from the one-launch kernel; larger ones are compacted by K5 through a plan
    ONE_CELLS = 48 * 1024

    def query(self, q: QuerySpec, agg) -> None:
        """One query through cs_query_one (K8 latency class: one launch, descriptor as a kernel
        parameter, results in mapped host memory; larger queries take the one-shot batch path
        inside the library): fused scalars for NullSink / LogLikelihood / MdlScore /
        MutualInformation, the dense table compacted on the host for small tables, the K5
        device compaction otherwise."""
        q.validate(self.db)
        kind = _fusion_kind(agg)
        vs = _vars(q)
        ar = self.gdb.arities
        if kind is not None:
            # per-thread scratch with cached addresses: no numpy / ctypes helper objects per call
            sc = self._tls.__dict__.get("one")
            if sc is None or len(sc[0]) < len(vs):
                vb = np.zeros(max(64, len(vs)), dtype=np.int32)
                ob = np.zeros(3)
                sc = self._tls.one = (vb, ob, vb.ctypes.data, ob.ctypes.data)
            vb, ob, va, oa = sc
            vb[:len(vs)] = vs
            N.check(N.lib.cs_query_one(self.gdb.handle, len(vs), va, 0, None, oa,
                                       oa + 8 if kind == "mi" else None, oa + 16))
            _absorb(agg, kind, float(ob[0]), float(ob[1]), int(ob[2:3].view(np.int64)[0]))
            return
        cells = 1
        for v in vs:
            cells *= int(ar[v])
        got = None
        if cells <= min(self.ONE_CELLS, _dense_limit()) and len(vs) <= 8:
            # the record stream straight from the single-query kernel (cell order), or
            # CS_ERR_UNSUPPORTED when the query is outside its class
            sc = self._tls.__dict__.get("cells")
            if sc is None:
                bufs = np.zeros((3, self.ONE_CELLS), dtype=np.int64)
                nz = np.zeros(1, dtype=np.int64)
                vb = np.zeros(8, dtype=np.int32)
                sc = self._tls.cells = (bufs, nz, vb, bufs[0].ctypes.data, bufs[1].ctypes.data,
                                        bufs[2].ctypes.data, nz.ctypes.data, vb.ctypes.data)
            bufs, nz, vb, a0, a1, a2, an, va = sc
            vb[:len(vs)] = vs
            rc = N.lib.cs_query_one_cells(self.gdb.handle, len(vs), va, a0, a1, a2, an)
            if rc == N.CS_OK:
                n = int(nz[0])
                got = (bufs[0, :n], bufs[1, :n].copy(), bufs[2, :n].copy())
            elif rc != N.CS_ERR_UNSUPPORTED:
                N.check(rc)
        if got is None:
            with self._lock:
                plan = QueryPlan(self.gdb, [vs], N.CS_WANT_TABLES)
                nnz = np.zeros(1, dtype=np.int64)
                plan.execute(nnz=nnz)
                _, cidx, nijk, nij = plan.compact(None, nnz)
                plan.close()
            got = (cidx, nijk, nij)
        self._deliver(q, agg, *got)

    def _deliver(self, q: QuerySpec, agg, cidx, nijk, nij) -> None:
        if not getattr(agg, "wants_records", False):
            agg.accept_block(nijk, nij)
            return
        ar = self.db.arities
        r_t = int(ar[q.target])
        parents = q.parents
        js = cidx // r_t
        # each parent's state of every record, vectorised (cell = k + r_t (s_p0 + r_p0 (s_p1 ...)))
        states = {}
        stride = 1
        for p in parents:
            r = int(ar[p])
            states[p] = ((js // stride) % r).tolist()
            stride *= r
        ordered = sorted(parents)
        configs = zip(*[zip(itertools.repeat(p), states[p]) for p in ordered]) if parents else \
            itertools.repeat((), len(js))
        accept = agg.accept_record
        for cfg, k, x, n in zip(configs, (cidx % r_t).tolist(), nijk.tolist(), nij.tolist()):
            accept(cfg, k, x, n)

    def count(self, a: Assignment) -> int:
        a.validate(self.db)
        with self._lock:
            return int(self.gdb.count_points([(a.variables, a.states)])[0])

    # -- batched API ------------------------------------------------------------------------
    def query_batch(self, queries, loglik: bool = True, mi: bool = False, nnz: bool = False,
                    tables: bool = False) -> dict:
        """Run many QuerySpecs in one launch; returns numpy arrays keyed by output name.

        Without ``tables`` the batch goes through the one-shot ``cs_query_batch`` (transient
        plan buffers; big batches plan chunk j+1 while chunk j runs) and ``cells`` /
        ``table_off`` are None; with ``tables`` a QueryPlan also reports each table's layout.
        """
        qs = list(queries)
        enc = _encode_specs(qs) if qs else None
        self._validate_encoded(qs, enc)
        if not tables:
            ll = np.zeros(len(qs)) if loglik else None
            mv = np.zeros(len(qs)) if mi else None
            nz = np.zeros(len(qs), dtype=np.int64) if nnz else None
            if qs:
                off, flat = enc
                with self._lock:
                    self.gdb.query_batch(off, flat, 0, loglik=ll, mi=mv, nnz=nz)
            return {"loglik": ll, "mi": mv, "nnz": nz, "tables": None, "cells": None, "table_off": None}
        with self._lock:
            plan = QueryPlan(self.gdb, enc if qs else [], N.CS_WANT_TABLES if tables else 0)
            out = {}
            ll = np.zeros(len(qs)) if loglik else None
            mv = np.zeros(len(qs)) if mi else None
            nz = np.zeros(len(qs), dtype=np.int64) if nnz else None
            tb = np.zeros(plan.total_cells, dtype=np.uint32) if tables else None
            if qs:
                plan.execute(tables=tb, loglik=ll, mi=mv, nnz=nz)
            out.update({"loglik": ll, "mi": mv, "nnz": nz, "tables": tb,
                        "cells": plan.cells, "table_off": plan.table_off})
            plan.close()
        return out

    def _validate_encoded(self, qs, enc) -> None:
        """QuerySpec.validate (variable < n; construction already checked the rest) for a whole
        batch with one vectorised test; on failure the per-query loop raises the reference's
        error for the first offending query."""
        if enc is None:
            return
        if len(enc[1]) and int(enc[1].max()) >= self.db.n:
            for q in qs:
                q.validate(self.db)

    def family_scores(self, families) -> tuple[np.ndarray, np.ndarray]:
        """(LL, MDL) of many (target, parents) families from one launch over their distinct
        variable subsets (see engine.FamilyScorer)."""
        fams = [(int(t), tuple(ps)) for t, ps in families]
        for t, ps in fams:
            QuerySpec(t, ps).validate(self.db)
        with self._lock:
            fs = FamilyScorer(self.gdb, fams, m_total=self.db.m)
            out = fs.scores()
            fs.plan.close()
        return out

    def count_batch(self, assignments) -> np.ndarray:
        al = list(assignments)
        for a in al:
            a.validate(self.db)
        with self._lock:
            return self.gdb.count_points([(a.variables, a.states) for a in al])


def make_strategies(db, names=STRATEGY_NAMES, adtree_leaf_threshold=None, adtree_node_cap=None,
                    device: int = 0):
    """Build the named strategies, timing each build (harness.py:125-158).

    Structural build failures (the device cannot hold the database, arity
    above 256) are reported in the failures mapping instead of aborting.
    """
    if isinstance(names, str):
        names = (names,)
    built, failures = {}, {}
    for name in names:
        t0 = time.perf_counter()
        if name not in STRATEGY_NAMES:
            hint = (" (a CPU engine of the reference package; this engine is 'gpu')"
                    if name in REFERENCE_CPU_STRATEGIES else "")
            raise ValueError(f"unknown strategy {name!r}{hint}; choose from {STRATEGY_NAMES}")
        try:
            s = GpuStrategy(db, device=device)
        except (N.EngineError, ValueError) as e:
            if isinstance(e, InvalidQueryError):
                raise
            failures[name] = str(e)
            continue
        s.build_seconds = time.perf_counter() - t0
        built[name] = s
    return built, failures


# ---------------------------------------------------------------------------------------------
# random-query benchmark (harness.py:161-275)


@dataclass(frozen=True)
class RandomQueryStream:
    """Reproducible random queries (harness.py:165-194): target uniform, |Pa| uniform on
    [1, n-1], parents without replacement; Philox keyed by SeedSequence(seed, spawn_key=(1,))."""

    seed: int
    count: int
    queries: tuple

    @classmethod
    def generate(cls, n: int, count: int, seed: int) -> "RandomQueryStream":
        if n < 2:
            raise ValueError(f"random queries need n >= 2 variables, got n={n}")
        g = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=(1,))))
        out = []
        for _ in range(count):
            t = int(g.integers(0, n))
            size = int(g.integers(1, n))
            rest = [v for v in range(n) if v != t]
            pick = g.choice(len(rest), size=size, replace=False)
            out.append(QuerySpec(t, tuple(rest[i] for i in sorted(pick))))
        return cls(seed, count, tuple(out))


@dataclass
class TimingRecord:
    query_id: int
    strategy: str
    pa_size: int
    durations_us: tuple
    record_count: int
    timed_out: bool = False

    @property
    def mean_us(self) -> float:
        return sum(self.durations_us) / len(self.durations_us)


@dataclass
class BenchResult:
    stream: RandomQueryStream
    timings: list
    build_seconds: dict
    build_failures: dict

    def by_strategy(self, name: str) -> list:
        return [t for t in self.timings if t.strategy == name]


def _time_query(strategy, q, repetitions, timeout_s):
    durations = []
    sink = NullSink()
    for _ in range(repetitions):
        sink = NullSink()
        t0 = time.perf_counter()
        strategy.query(q, sink)
        durations.append((time.perf_counter() - t0) * 1e6)
        if timeout_s is not None and durations[-1] > timeout_s * 1e6:
            return durations, sink.count, True
    return durations, sink.count, False


def bench_random(db, num_queries: int = 100, seed: int = 0, strategies=STRATEGY_NAMES,
                 repetitions: int = 5, timeout_s=None, parallel: int = 1,
                 adtree_leaf_threshold=None, adtree_node_cap=None) -> BenchResult:
    """Time each strategy on one shared random stream (harness.py:235-275)."""
    stream = RandomQueryStream.generate(db.n, num_queries, seed)
    built, failures = make_strategies(db, strategies)
    jobs = [(qid, q, name) for qid, q in enumerate(stream.queries) for name in built]

    def run(job):
        qid, q, name = job
        d, rc, to = _time_query(built[name], q, repetitions, timeout_s)
        return TimingRecord(qid, name, len(q.parents), tuple(d), rc, to)

    if parallel > 1:
        with ThreadPoolExecutor(max_workers=parallel) as ex:
            timings = list(ex.map(run, jobs))
    else:
        timings = [run(j) for j in jobs]
    return BenchResult(stream, timings, {k: s.build_seconds for k, s in built.items()}, failures)


# ---------------------------------------------------------------------------------------------
# MDL parent-set selection (harness.py:282-348)


@dataclass
class ParentSetResult:
    target: int
    parents: tuple
    score: float
    candidates_scored: int
    query_seconds: float
    wall_seconds: float

    @property
    def query_fraction(self) -> float:
        return self.query_seconds / self.wall_seconds if self.wall_seconds > 0 else 0.0


def candidate_parent_sets(n: int, target: int, max_parents: int):
    """Reference enumeration order: size ascending, itertools.combinations (harness.py:316-322)."""
    others = [v for v in range(n) if v != target]
    for size in range(max_parents + 1):
        yield from itertools.combinations(others, size)


def _argmin_mdl(combos, scores, tie_eps):
    """Sequential argmin with the reference's relative tie rule (harness.py:330-337)."""
    best_score, best_set = None, None
    for combo, score in zip(combos, scores):
        score = float(score)
        if best_score is None:
            best_score, best_set = score, combo
            continue
        eps = tie_eps * (1.0 + abs(best_score))
        if score < best_score - eps:
            best_score, best_set = score, combo
        elif abs(score - best_score) <= eps and combo < best_set:
            best_set = combo
    return best_score, best_set


def mdl_penalties(db, target: int, combos) -> np.ndarray:
    ar = db.arities
    r_i = int(ar[target])
    lnm = math.log(db.m)
    out = np.empty(len(combos))
    for i, c in enumerate(combos):
        q_i = 1
        for p in c:
            q_i *= int(ar[p])
        out[i] = 0.5 * lnm * (r_i - 1) * q_i
    return out


def learn_parents(db, strategy, max_parents: int = 3, tie_eps: float = 1e-9) -> list:
    """Exhaustive MDL parent sets up to ``max_parents`` per target (harness.py:296-348).

    With a batched strategy every target's candidates go to the device as one
    batch; scores are MdlScore's formula on the fused LL and the argmin uses
    the reference's enumeration order and tie rule, so the result is
    strategy-invariant.  Any other strategy is driven one query at a time.
    """
    if max_parents < 0 or max_parents > db.n - 1:
        raise ValueError(f"max_parents must be in [0, n-1], got {max_parents}")
    results = []
    if hasattr(strategy, "family_scores"):
        # every target's candidates in one device batch over the distinct variable subsets
        t_all = time.perf_counter()
        cand = [list(candidate_parent_sets(db.n, t, max_parents)) for t in range(db.n)]
        fams = [(t, c) for t in range(db.n) for c in cand[t]]
        t0 = time.perf_counter()
        _, mdl = strategy.family_scores(fams)
        qsec = time.perf_counter() - t0
        wall = time.perf_counter() - t_all
        pos = 0
        for t in range(db.n):
            k = len(cand[t])
            best_score, best_set = _argmin_mdl(cand[t], mdl[pos:pos + k], tie_eps)
            pos += k
            share = k / max(len(fams), 1)
            results.append(ParentSetResult(t, best_set, best_score, k, qsec * share, wall * share))
        return results
    batched = hasattr(strategy, "query_batch")
    for target in range(db.n):
        t_wall = time.perf_counter()
        combos = list(candidate_parent_sets(db.n, target, max_parents))
        if batched:
            t0 = time.perf_counter()
            ll = strategy.query_batch([QuerySpec(target, c) for c in combos], loglik=True)["loglik"]
            qsec = time.perf_counter() - t0
            scores = -ll + mdl_penalties(db, target, combos)
        else:
            scores = []
            qsec = 0.0
            for c in combos:
                q = QuerySpec(target, c)
                agg = MdlScore.for_query(db, q)
                t0 = time.perf_counter()
                strategy.query(q, agg)
                qsec += time.perf_counter() - t0
                scores.append(agg.result())
        best_score, best_set = _argmin_mdl(combos, scores, tie_eps)
        results.append(ParentSetResult(target, best_set, best_score, len(combos), qsec,
                                       time.perf_counter() - t_wall))
    return results


# ---------------------------------------------------------------------------------------------
# association-rule mining (harness.py:351-429)


@dataclass(frozen=True, order=True)
class AssociationRule:
    antecedent: tuple
    consequent: int
    support: float
    confidence: float


def mine_rules(db, strategy, min_support: float = 0.2, min_confidence: float = 0.3,
               max_size: int = 6) -> set:
    """Level-wise frequent itemsets + rules on a binary database (harness.py:365-429).

    Each apriori level's candidate supports are one ``count_batch`` call when
    the strategy has it (one device launch per level).
    """
    if (np.asarray(db.arities) != 2).any():
        raise ValueError(
            "association-rule mining needs a binary database; "
            f"arities are {np.asarray(db.arities).tolist()}"
        )
    if min_support <= 0 or min_confidence <= 0:
        raise ValueError("thresholds must be positive")
    if max_size < 2:
        raise ValueError(f"max_size must be >= 2, got {max_size}")

    def supports(itemsets):
        if not itemsets:
            return []
        if hasattr(strategy, "count_batch"):
            c = strategy.count_batch([Assignment(s, (1,) * len(s)) for s in itemsets])
            return [int(x) / db.m for x in c]
        return [strategy.count(Assignment(s, (1,) * len(s))) / db.m for s in itemsets]

    support = {}
    singles = [(v,) for v in range(db.n)]
    level = []
    for s, val in zip(singles, supports(singles)):
        if val >= min_support:
            support[s] = val
            level.append(s)
    size = 1
    while level and size < max_size:
        size += 1
        prev = set(level)
        cands = set()
        for a, b in itertools.combinations(sorted(level), 2):
            if a[:-1] != b[:-1]:
                continue
            c = a + (b[-1],)
            if all(c[:i] + c[i + 1:] in prev for i in range(len(c))):
                cands.add(c)
        ordered = sorted(cands)
        level = []
        for c, val in zip(ordered, supports(ordered)):
            if val >= min_support:
                support[c] = val
                level.append(c)
    rules = set()
    for itemset, s in support.items():
        if len(itemset) < 2:
            continue
        for i, cons in enumerate(itemset):
            ant = itemset[:i] + itemset[i + 1:]
            conf = s / support[ant]
            if conf >= min_confidence:
                rules.add(AssociationRule(ant, cons, s, conf))
    return rules
