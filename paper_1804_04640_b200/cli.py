"""Command-line front end with the reference's interface and JSONL schema (reference cli.py).

    python -m paper_1804_04640_b200 {query,bench-random,learn-parents,mine-rules} ...

Same subcommands, flags, record types (`build`, `build_failure`, `record`, `score`, `timing`,
`strategy_summary`, `layer_summary`, `parent_set`, `rule`, `warning`, `summary`), CSV mode and
exit codes (0 ok, 1 data error / failed build, 2 usage) as the reference CLI (cli.py:1-12,
114-331), with the B200 engine registered as strategy ``gpu`` (the default).  A client of the
reference CLI -- e.g. its TypeScript subprocess bindings -- can point at this module instead.
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
import time

import numpy as np

from .aggregators import LogLikelihood, MdlScore, RecordCollector
from .database import DatabaseLoadError, InvalidQueryError, QuerySpec, load_arities, load_csv, parse_synthetic
from .harness import STRATEGY_NAMES, bench_random, learn_parents, make_strategies, mine_rules

__all__ = ["main", "build_parser"]


class JsonlOrCsv:
    """One self-describing JSON object per line, or CSV rows of a single record type."""

    def __init__(self, fh, fmt: str, csv_type: str):
        self.fh, self.fmt, self.csv_type = fh, fmt, csv_type
        self.writer = None

    def __call__(self, **fields):
        if self.fmt == "jsonl":
            self.fh.write(json.dumps(fields) + "\n")
            return
        if fields.get("type") != self.csv_type:
            return
        row = {k: (" ".join(map(str, v)) if isinstance(v, (list, tuple)) else v)
               for k, v in fields.items() if k != "type"}
        if self.writer is None:
            self.writer = csv.DictWriter(self.fh, fieldnames=list(row))
            self.writer.writeheader()
        self.writer.writerow(row)


def database_from_args(a):
    if a.synthetic and a.input:
        raise ValueError("--input and --synthetic are mutually exclusive")
    if a.synthetic:
        return parse_synthetic(a.synthetic, a.seed)
    if not a.input:
        raise ValueError("one of --input or --synthetic is required")
    ar = load_arities(a.arities) if a.arities else None
    if getattr(a, "device_ingest", False):
        from .harness import load_csv_device  # tokenise on the GPU (cs_db_load_text)

        return load_csv_device(a.input, delimiter=a.delimiter, arities=ar)
    return load_csv(a.input, delimiter=a.delimiter, arities=ar)


def strategy_list(text: str) -> tuple:
    if text == "all":
        return STRATEGY_NAMES
    names = tuple(x.strip() for x in text.split(",") if x.strip())
    if not names:
        raise ValueError("no strategies given")
    bad = [x for x in names if x not in STRATEGY_NAMES]
    if bad:
        raise ValueError(f"unknown strategy {bad[0]!r}; choose from {', '.join(STRATEGY_NAMES)} or 'all'")
    return names


def build_one(db, name, emit):
    built, failed = make_strategies(db, (name,))
    for n, s in built.items():
        emit(type="build", strategy=n, seconds=s.build_seconds)
    for n, err in failed.items():
        emit(type="build_failure", strategy=n, error=err)
    return built.get(name)


def run_query(a, emit) -> int:
    db = database_from_args(a)
    parents = tuple(int(x) for x in a.parents.split(",") if x.strip()) if a.parents else ()
    q = QuerySpec(a.target, parents)
    q.validate(db)
    s = build_one(db, a.strategy, emit)
    if s is None:
        return 1
    if a.agg == "records":
        col = RecordCollector()
        s.query(q, col)
        recs = sorted(col.result())
        for r in recs:
            emit(type="record", config=[list(p) for p in r.config], k=r.k, n_ijk=r.n_ijk, n_ij=r.n_ij)
        emit(type="summary", records=len(recs))
        return 0
    agg = LogLikelihood() if a.agg == "loglik" else MdlScore.for_query(db, q)
    s.query(q, agg)
    emit(type="score", name=a.agg, value=agg.result())
    return 0


def run_bench_random(a, emit) -> int:
    db = database_from_args(a)
    res = bench_random(db, num_queries=a.queries, seed=a.seed, strategies=strategy_list(a.strategies),
                       repetitions=a.repetitions,
                       timeout_s=a.timeout_ms / 1000 if a.timeout_ms else None, parallel=a.parallel)
    for n, sec in res.build_seconds.items():
        emit(type="build", strategy=n, seconds=sec)
    for n, err in res.build_failures.items():
        emit(type="build_failure", strategy=n, error=err)
    for t in res.timings:
        emit(type="timing", query_id=t.query_id, strategy=t.strategy, pa_size=t.pa_size, mean_us=t.mean_us,
             durations_us=list(t.durations_us), records=t.record_count, timed_out=t.timed_out)
    for n in res.build_seconds:
        rows = res.by_strategy(n)
        if not rows:
            continue
        means = np.array([t.mean_us for t in rows])
        emit(type="strategy_summary", strategy=n, queries=len(rows), mean_us=float(means.mean()),
             median_us=float(np.median(means)), p95_us=float(np.percentile(means, 95)),
             timeouts=sum(t.timed_out for t in rows))
        for pa in sorted({t.pa_size for t in rows}):
            layer = [t.mean_us for t in rows if t.pa_size == pa]
            emit(type="layer_summary", strategy=n, pa_size=pa, queries=len(layer), mean_us=float(np.mean(layer)))
    return 0


def run_learn_parents(a, emit) -> int:
    db = database_from_args(a)
    s = build_one(db, a.strategy, emit)
    if s is None:
        return 1
    res = learn_parents(db, s, max_parents=a.max_parents)
    for r in res:
        emit(type="parent_set", target=r.target, parents=list(r.parents), score=r.score,
             candidates=r.candidates_scored, query_seconds=r.query_seconds, wall_seconds=r.wall_seconds,
             query_fraction=r.query_fraction)
    wall = sum(r.wall_seconds for r in res)
    qs = sum(r.query_seconds for r in res)
    emit(type="summary", targets=len(res), candidates=sum(r.candidates_scored for r in res),
         query_seconds=qs, wall_seconds=wall, query_fraction=qs / wall if wall else 0.0)
    return 0


def run_mine_rules(a, emit) -> int:
    db = database_from_args(a)
    if a.min_support > 1 or a.min_confidence > 1:
        emit(type="warning", message="threshold above 1: no itemset can qualify, rule set will be empty")
    s = build_one(db, a.strategy, emit)
    if s is None:
        return 1
    t0 = time.perf_counter()
    rules = mine_rules(db, s, min_support=a.min_support, min_confidence=a.min_confidence, max_size=a.max_size)
    sec = time.perf_counter() - t0
    for r in sorted(rules, key=lambda r: (len(r.antecedent), r.antecedent, r.consequent)):
        emit(type="rule", antecedent=list(r.antecedent), consequent=r.consequent, support=r.support,
             confidence=r.confidence)
    emit(type="summary", rules=len(rules), seconds=sec)
    return 0


def _db_flags(p):
    p.add_argument("--input", help="delimited text file of integer states, one record per line")
    p.add_argument("--delimiter", default=None, help="field delimiter (default: any whitespace)")
    p.add_argument("--arities", help="sidecar file declaring one arity per variable")
    p.add_argument("--device-ingest", action="store_true",
                   help="parse --input on the GPU (same grammar and errors; the data never exists on the host)")
    p.add_argument("--synthetic", metavar="n=..,m=..,arity=..", help="generate a uniform random database")
    p.add_argument("--seed", type=int, default=0, help="seed for synthetic data and query streams (default 0)")
    p.add_argument("--adtree-leaf", type=int, default=None, help="accepted for compatibility (unused)")
    p.add_argument("--adtree-node-cap", type=int, default=None, help="accepted for compatibility (unused)")
    p.add_argument("--out", default=None, help="output path (default: stdout)")
    p.add_argument("--format", choices=("jsonl", "csv"), default="jsonl")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="countstream-b200",
                                 description="Counting queries over categorical data on B200.")
    sub = ap.add_subparsers(dest="command", required=True)
    specs = [
        ("bench-random", "time strategies on a random query stream", run_bench_random, "timing"),
        ("learn-parents", "select MDL-optimal parent sets per variable", run_learn_parents, "parent_set"),
        ("mine-rules", "mine association rules from a binary database", run_mine_rules, "rule"),
        ("query", "run one counting query", run_query, "record"),
    ]
    for name, helptext, fn, csv_type in specs:
        p = sub.add_parser(name, help=helptext)
        _db_flags(p)
        p.set_defaults(func=fn, csv_type=csv_type)
        if name == "bench-random":
            p.add_argument("--queries", type=int, default=100)
            p.add_argument("--repetitions", type=int, default=5)
            p.add_argument("--strategies", default="all")
            p.add_argument("--timeout-ms", type=float, default=None)
            p.add_argument("--parallel", type=int, default=1)
        elif name == "learn-parents":
            p.add_argument("--max-parents", type=int, default=3)
            p.add_argument("--strategy", default="gpu", choices=STRATEGY_NAMES)
        elif name == "mine-rules":
            p.add_argument("--min-support", type=float, default=0.2)
            p.add_argument("--min-confidence", type=float, default=0.3)
            p.add_argument("--max-size", type=int, default=6)
            p.add_argument("--strategy", default="gpu", choices=STRATEGY_NAMES)
        else:
            p.add_argument("--target", type=int, required=True)
            p.add_argument("--parents", default="")
            p.add_argument("--strategy", default="gpu", choices=STRATEGY_NAMES)
            p.add_argument("--agg", default="records", choices=("records", "loglik", "mdl"))
    return ap


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    fh = open(a.out, "w", newline="") if a.out else sys.stdout
    try:
        return a.func(a, JsonlOrCsv(fh, a.format, a.csv_type))
    except (DatabaseLoadError, InvalidQueryError, ValueError, OSError) as e:
        sys.stderr.write(json.dumps({"type": "error", "message": str(e)}) + "\n")
        return 1
    finally:
        if a.out:
            fh.close()
