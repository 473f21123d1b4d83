#!/usr/bin/env python3
"""Benchmark: batched counting queries on B200 (BASELINE.json metric: count queries/s and
scanned GB/s vs HBM peak), one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]

Default workload is BASELINE configs[1] (cfg2: n=100 variables, arity U{2..5}, Dirichlet(1)
marginals, m=1e6 uint8 instances, 10,000 queries of 1..6 variables, joint tables out) -- the
config BASELINE's metric is quoted on that fits one GPU.  A step = the whole query batch.
Other configs (--config cfg1|cfg3|cfg4|cfg5) measure the remaining BASELINE workloads.

Multi-GPU (torchrun, one rank per GPU, NCCL):
  cfg1-cfg4  query sharding: each rank runs its own slice of an N x batch (weak scaling).
  cfg5       instance sharding: rank g holds rows [g m/N, (g+1) m/N); partial N_ijk tables
             are reduce-scattered to their owners over NCCL (CS_BENCH_MERGE=allreduce: summed
             on every rank), owners score LL + MI, scores all-gathered (strong scaling).

value      units/s over all ranks, device-timed (CUDA events on the launch stream, max over
           ranks), database + plan resident in HBM; L2 flushed (256 MB write) before every
           timed step.
e2e        through the C ABI with HOST buffers each step: query descriptors in, tables /
           scores / supports out to pinned host memory.
roofline   the dominant kernel (k_hist, or k_itemsets for cfg4): algorithmic bytes per launch
            / its device time (library CUDA events, same stream).
cpu_baseline  the oracle's C restatement of the reference path (port, all host threads, and
           one core) on a bounded sample of the same workload.
--impl reference  times that CPU port on all host threads (`value`) and on one core, plus the
           reference itself -- countstream's numba RadixStrategy, installed unmodified in the
           git-ignored baseline/_ref -- as forked processes and on one core (DESIGN.md
           "Reference arm").  libcountgpu.so is never mapped into that process.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "count queries/s"
UNIT = "queries/s"
L2_FLUSH_BYTES = 256 << 20


def load_peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(config: str):
    """dram read+write bytes per launch of the dominant kernel, from the committed ncu capture."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get(config)
        except Exception:
            return None
    return None


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, device: int, period_s: float = 0.005):
        self.period = period_s
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self._t = None
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def load_l2_peak() -> tuple[float, str]:
    """L2 -> SM streaming ceiling (GB/s): MEASURED_PEAKS has no L2 figure, so it comes from the
    committed microbenchmark output (tools/microbench2.cu, profiles/ceilings.json)."""
    p = ROOT / "profiles" / "ceilings.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["l2_to_sm_gbs"]), d.get("l2_source", "profiles/ceilings.json")
        except Exception:
            pass
    return 11_800.0, "tools/microbench2.cu ld.global.nc.v4 L2->SM, upper end of the 9.5-11.8 TB/s range (DESIGN.md)"


def layout_bytes_per_row(arities) -> float:
    """Bytes per row of the column copy the histogram kernels read: the
    2-bit copy when every arity <= 4, the 4-bit copy when every arity <= 16, else uint8."""
    a = int(np.max(arities))
    return 0.25 if a <= 4 else 0.5 if a <= 16 else 1.0


def counting_roofline(r, k_ms: float) -> dict:
    """Roofline of the histogram phase (K1 / K1r launches of one step; library CUDA events).

    input_bytes = sum over queries of k x rows x (bytes per row of the column copy read).  The
    databases of cfg1-cfg3 (<= 100 MB of columns) stay L2-resident across the batch, so their
    bound is the L2 -> SM stream (measured ceiling); cfg5's 50 GB 4-bit copy cannot, so its bound
    is HBM.  The `hbm` object gives the HBM view for every config: survey 8(d)'s logical bytes
    (uint8, k x m per query) and the DRAM bytes ncu measured for the same launches."""
    peak_hbm, src_hbm = load_peaks()
    bpr = layout_bytes_per_row(r.w.arities)
    input_bytes = r.algo_bytes * bpr
    ks = k_ms / 1e3
    traffic = load_traffic(r.config)
    if traffic is None and r.config == "cfg5":
        per_q = load_traffic("cfg5_per_query")
        traffic = per_q * r.units * (r.rows / r.w.m) if per_q else None  # rows: this rank's shard
    hbm = {"peak": peak_hbm, "peak_source": src_hbm, "logical_bytes": r.algo_bytes,
           "logical_frac": r.algo_bytes / ks / 1e9 / peak_hbm,
           "dram_bytes": traffic, "dram_frac": (traffic / ks / 1e9 / peak_hbm) if traffic else None}
    if r.config == "cfg5":
        bound, peak, src = "hbm", peak_hbm, src_hbm
    else:
        bound, (peak, src) = "l2", load_l2_peak()
    achieved = input_bytes / ks / 1e9
    return {"bound": bound, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": r.kernel, "kernel_ms": k_ms, "peak_source": src,
            "input_bytes": input_bytes, "bytes_per_row": bpr, "hbm": hbm,
            "note": "achieved = bytes of the column copy the kernels read (k x rows x bytes_per_row per "
                    "query) / histogram-phase time; traffic = ncu dram read+write of the same launches "
                    "(profiles/traffic.json)"}


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O  # test infrastructure: only the cpu_baseline / reference legs use it

    return O


def _twin():
    sys.path.insert(0, str(ROOT / "oracle"))
    import gen_twin

    return gen_twin


def host_columns(w, variables=None, rows=None):
    """Workload columns on the host for the CPU legs (reference generator or numpy twin)."""
    if w.host_db is not None:
        u8 = w.host_db.columns_u8()
        return u8 if variables is None else u8[list(variables)]
    rows = np.arange(w.m, dtype=np.int64) if rows is None else rows
    vs = list(range(w.n)) if variables is None else list(variables)
    cols = _twin().generate_workload_columns(w, rows, vs)
    return np.vstack([cols[v] for v in vs])


# ---------------------------------------------------------------------------------------------
# workloads


OUTPUTS = {"cfg1": "tables+loglik", "cfg2": "tables", "cfg3": "loglik+mdl", "cfg4": "pair+triple supports",
           "cfg5": "loglik+mi"}
L2_NOTE = ("GPU arm: L2 NOT flushed (CS_BENCH_NOFLUSH=1, diagnostic run)" if os.environ.get("CS_BENCH_NOFLUSH") == "1"
           else "GPU arm: L2 flushed (256 MB write) before every timed step")


def arm_config(config: str, w, units: int) -> dict:
    """The `config` object both arms print (identical, so the driver can pair them)."""
    unit = {"cfg3": "families_per_step", "cfg4": "itemsets_per_step"}.get(config, "queries_per_step")
    return {"workload": config, "n": int(w.n), "m": int(w.m), unit: int(units), "outputs": OUTPUTS[config],
            "l2": L2_NOTE}


def workload(config: str, world: int, rank: int, nq_override):
    """(Workload, this rank's query list) for the query configs."""
    from paper_1804_04640_b200 import workloads as W

    if config == "cfg1":
        w = W.cfg1(nq=(nq_override or 1000) * world)
    elif config == "cfg2":
        w = W.cfg2(nq=(nq_override or 10_000) * world)
        kf = os.environ.get("CS_BENCH_KFILTER")  # diagnostic: only queries with k variables
        if kf:
            w.queries = [q for q in w.queries if len(q) == int(kf)]
    elif config == "cfg3":
        w = W.cfg3()
        if nq_override:
            w.queries = w.queries[: nq_override * world]
        return w, w.queries[rank::world]
    elif config == "cfg5":
        w = W.cfg5(nq=nq_override or 100_000)  # BASELINE configs[4]: the 100,000-query stream
        return w, w.queries  # instance sharded: every rank runs every query on its rows
    else:
        raise SystemExit(f"unsupported --config {config}")
    per = len(w.queries) // world
    return w, w.queries[rank * per:(rank + 1) * per]


def cpu_rate_queries(w, queries, budget_s, threads, row_limit=None, cols_fn=None):
    """Oracle port (radix restatement) on a bounded sample of `queries`; q/s scaled to full m.

    cols_fn(vars, nrows) supplies host columns (default: the reference generator / numpy twin);
    building them is not timed.
    """
    O = _oracle()
    rows = None if row_limit is None or row_limit >= w.m else np.arange(row_limit, dtype=np.int64)
    m_eff = w.m if rows is None else len(rows)

    def timed(qs):
        vs = sorted({v for q in qs for v in q})
        cols = cols_fn(vs, m_eff) if cols_fn else host_columns(w, vs, rows)
        remap = {v: i for i, v in enumerate(vs)}
        ar = np.asarray([w.arities[v] for v in vs])
        t0 = time.perf_counter()
        O.radix_tables(cols, ar, [tuple(remap[v] for v in q) for q in qs], nthreads=threads,
                       want_tables=False)
        return time.perf_counter() - t0

    probe = list(queries[: max(2 * threads, 16)])
    rate = len(probe) / max(timed(probe), 1e-6)
    n = int(max(len(probe), rate * budget_s))
    reps = max(1, -(-n // len(queries)))  # small batches (cfg1) are repeated to fill the budget
    sample = (list(queries) * reps)[:n]
    dt = timed(sample)
    scale = m_eff / w.m  # radix work is linear in m
    desc = (f"{n} {w.name} queries (of a {len(queries)}-query batch) in {dt:.1f} s "
            f"(oracle/radix_oracle.c radix restatement, {threads} threads"
            + (f", on the first {m_eff} rows, rate scaled x{scale:g} to m={w.m}" if rows is not None else "")
            + ")")
    return n / dt * scale, desc


class QueryRunner:
    """cfg1/cfg2/cfg3 (query-sharded) and cfg5 (instance-sharded + NCCL merge)."""

    kernel = "k_hist"

    def __init__(self, args, world, rank, local, torch, ctx):
        from paper_1804_04640_b200 import _native as N
        from paper_1804_04640_b200.engine import QueryPlan, encode_queries

        self.torch, self.ctx, self.world, self.rank = torch, ctx, world, rank
        self.config = args.config
        self.w, self.queries = workload(args.config, world, rank, args.nq)
        w = self.w
        if args.config == "cfg5":
            self.kernel = "k_hist + k_spill_hist + k_spill_count + k_radix_part + k_radix_count (histogram phase)"
        # CS_BENCH_FORCE_SHARDED=1 runs the instance-sharded path (CS_PARTIAL + NCCL all-reduce
        # + cs_plan_score) even at world size 1 -- exercises it on a single-GPU box
        self.sharded = args.config == "cfg5" and (world > 1 or os.environ.get("CS_BENCH_FORCE_SHARDED") == "1")
        t0 = time.perf_counter()
        if self.sharded:
            from paper_1804_04640_b200.parallel import shard_rows

            self.row0, self.rows = shard_rows(w.m, world, rank)
            self.gdb = w.build_device(ctx, row_offset=self.row0, m_shard=self.rows)
        else:
            self.rows = w.m
            self.gdb = w.build_device(ctx)
        ctx.sync()
        self.build_s = time.perf_counter() - t0
        self.want_tables = args.config in ("cfg1", "cfg2")
        self.want_ll = args.config in ("cfg1", "cfg3", "cfg5")
        self.want_mi = args.config == "cfg5"
        flags = N.CS_WANT_TABLES if self.want_tables else 0
        if self.sharded:
            flags |= N.CS_PARTIAL | N.CS_WANT_TABLES
        self.flags = flags
        # long streams (cfg5's 100,000 queries) run as consecutive plans of CHUNK queries sharing
        # one device table buffer: a step executes every plan (the whole stream)
        # (cfg5 only: the other configs' batches are one plan, as the reference-facing call is)
        chunk = int(os.environ.get("CS_BENCH_CHUNK", "2000")) if args.config == "cfg5" else 1 << 30
        self.chunks = []
        self.shard_runs = []
        self.merge = None
        cuts = list(range(0, len(self.queries), chunk)) + [len(self.queries)]
        if self.sharded:
            # instance sharding: consecutive CHUNK-query runners sharing one table buffer.
            # CS_BENCH_MERGE=reduce_scatter (default): partial tables reduce-scattered to their
            # owners, owners score, scores all-gathered; =allreduce: all-reduce, everyone scores
            from paper_1804_04640_b200 import parallel as PAR

            self.merge = os.environ.get("CS_BENCH_MERGE", "reduce_scatter")
            ar = w.arities
            cells = [[int(np.prod([int(ar[v]) for v in q], dtype=np.int64)) for q in self.queries[a:b]]
                     for a, b in zip(cuts[:-1], cuts[1:])]
            if self.merge == "allreduce":
                tb = torch.empty(max(sum(c) for c in cells), dtype=torch.int32, device="cuda")
                for a, b in zip(cuts[:-1], cuts[1:]):
                    self.shard_runs.append((a, b, PAR.InstanceShardedPlan(self.gdb, self.queries[a:b], tables=tb)))
            else:
                S = max(max(sum(c[i] for i in o) for o in PAR.owner_split(c, world)) for c in cells)
                buf = torch.zeros((world + 1) * (-(-S // 64) * 64), dtype=torch.int32, device="cuda")
                for a, b in zip(cuts[:-1], cuts[1:]):
                    self.shard_runs.append((a, b, PAR.ReduceScatterInstanceSharded(
                        self.gdb, self.queries[a:b], world, rank, buf=buf)))
            self.plan = self.shard_runs[0][2].plans[0] if self.merge != "allreduce" else self.shard_runs[0][2].plan
            self.kernel_is_step = True
        elif len(self.queries) > chunk:
            for c0, c1 in zip(cuts[:-1], cuts[1:]):
                self.chunks.append((c0, c1, QueryPlan(self.gdb, self.queries[c0:c1], flags)))
            self.plan = max((p for _, _, p in self.chunks), key=lambda p: p.total_cells)
            self.kernel_is_step = True  # the library's events bracket one plan; time the step
        else:
            self.plan = QueryPlan(self.gdb, self.queries, flags)
        self.units = len(self.queries)
        dev = "cuda"
        self.tables = (torch.empty(max(self.plan.total_cells, 1), dtype=torch.int32, device=dev)
                       if (self.want_tables or self.chunks) and not self.sharded else None)
        self.ll = torch.empty(self.units, dtype=torch.float64, device=dev) if self.want_ll else None
        self.mi = torch.empty(self.units, dtype=torch.float64, device=dev) if self.want_mi else None
        self.algo_bytes = float(sum(len(q) for q in self.queries)) * self.rows
        self.off, self.flat = encode_queries(self.queries)
        pin = dict(pin_memory=True)
        self.h_tables = (torch.empty(max(self.plan.total_cells, 1), dtype=torch.int32, **pin)
                         if self.want_tables else None)
        self.h_ll = torch.empty(self.units, dtype=torch.float64, **pin) if self.want_ll else None
        self.h_mi = torch.empty(self.units, dtype=torch.float64, **pin) if self.want_mi else None
        self.h2d = int(self.off.nbytes + self.flat.nbytes)
        self.d2h = int((self.plan.total_cells * 4 if self.want_tables else 0)
                       + self.units * 8 * (int(self.want_ll) + int(self.want_mi)))
        self.scaling = "strong" if self.sharded else "weak"
        self.parallelism = ((f"instance-shard x{world} + NCCL " +
                             ("all-reduce" if self.merge == "allreduce" else "reduce-scatter + owner scoring"))
                            if self.sharded else f"query-shard x{world}")

    def step(self):
        if self.sharded:
            for a, b, run in self.shard_runs:
                run.run(loglik=self.ll[a:b], mi=self.mi[a:b])
        elif self.chunks:
            for c0, c1, p in self.chunks:
                p.execute(tables=self.tables, loglik=None if self.ll is None else self.ll[c0:c1],
                          mi=None if self.mi is None else self.mi[c0:c1])
        else:
            self.plan.execute(tables=self.tables, loglik=self.ll, mi=self.mi)

    def e2e_step(self):
        if self.sharded:
            self.step()
            self.h_ll.copy_(self.ll)
            self.h_mi.copy_(self.mi)
            self.torch.cuda.synchronize()
            return
        if self.chunks:  # one-shot batches of the same chunks (bounded table scratch)
            for c0, c1, _ in self.chunks:
                o = self.off[c0:c1 + 1] - self.off[c0]
                self.gdb.query_batch(o, self.flat[self.off[c0]:self.off[c1]], self.flags,
                                     loglik=None if self.h_ll is None else self.h_ll[c0:c1],
                                     mi=None if self.h_mi is None else self.h_mi[c0:c1])
            return
        self.gdb.query_batch(self.off, self.flat, self.flags, tables=self.h_tables, loglik=self.h_ll,
                             mi=self.h_mi)

    def describe(self):
        return arm_config(self.config, self.w, self.units * (1 if self.sharded else self.world))

    def run_info(self):
        if self.chunks:
            return {"total_cells": int(sum(p.total_cells for _, _, p in self.chunks)),
                    "plans_per_step": len(self.chunks), "parallelism": self.parallelism}
        return {"total_cells": int(self.plan.total_cells), "parallelism": self.parallelism}

    def cpu_baseline(self, budget, threads):
        limit = 12_500_000 if self.w.m > 20_000_000 else None

        def cols_fn(vs, nrows):  # the very columns the GPU counted (download is untimed)
            return np.vstack([self.gdb.download(v, 0, nrows) for v in vs])

        return cpu_rate_queries(self.w, self.queries, budget, threads, row_limit=limit, cols_fn=cols_fn)


class FamilyRunner:
    """cfg3: MDL + LL of every (X_i, Pa), |Pa| <= 3 (288,859 families) via the N ln N sums of
    the 74,518 distinct variable subsets (one k_hist launch + k_family)."""

    kernel = "k_hist"

    def __init__(self, args, world, rank, local, torch, ctx):
        from paper_1804_04640_b200 import _native as N
        from paper_1804_04640_b200 import workloads as W
        from paper_1804_04640_b200.engine import FamilyScorer, encode_queries

        self.torch, self.ctx, self.world, self.rank = torch, ctx, world, rank
        self.config = "cfg3"
        self.N = N
        self.w = W.cfg3()
        w = self.w
        fams = [(q[0], tuple(q[1:])) for q in w.queries][rank::world]
        if args.nq:
            fams = fams[: args.nq]
        t0 = time.perf_counter()
        self.gdb = w.build_device(ctx)
        ctx.sync()
        self.build_s = time.perf_counter() - t0
        self.fs = FamilyScorer(self.gdb, fams)
        self.h_sidx, self.h_pidx, self.h_pen = self.fs.s_idx, self.fs.p_idx, self.fs.penalty
        self.fs.to_device(torch)
        self.units = self.fs.nfam
        self.nlogn = torch.empty(self.fs.nsub, dtype=torch.float64, device="cuda")
        self.ll = torch.empty(self.units, dtype=torch.float64, device="cuda")
        self.mdl = torch.empty(self.units, dtype=torch.float64, device="cuda")
        self.algo_bytes = float(sum(len(s) for s in self.fs.subsets)) * w.m
        self.family_bytes = float(sum(1 + len(p) for _, p in fams)) * w.m
        self.off, self.flat = encode_queries(self.fs.subsets)
        pin = dict(pin_memory=True)
        self.h_nlogn = torch.empty(self.fs.nsub, dtype=torch.float64, **pin)
        self.h_ll = torch.empty(self.units, dtype=torch.float64, **pin)
        self.h_mdl = torch.empty(self.units, dtype=torch.float64, **pin)
        self.h2d = int(self.off.nbytes + self.flat.nbytes + self.h_sidx.nbytes + self.h_pidx.nbytes
                       + self.h_pen.nbytes)
        self.d2h = int(self.units * 16 + self.fs.nsub * 8)
        self.scaling = "weak"
        self.parallelism = f"family-shard x{world}"

    def step(self):
        self.fs.run(self.nlogn, self.ll, self.mdl)

    def e2e_step(self):
        from paper_1804_04640_b200._native import check, lib, ptr

        self.gdb.query_batch(self.off, self.flat, self.N.CS_NLOGN, loglik=self.h_nlogn)
        check(lib.cs_family_scores(self.ctx.handle, self.units, ptr(self.h_nlogn), self.fs.nsub,
                                   ptr(self.h_sidx), ptr(self.h_pidx), ptr(self.h_pen), self.fs.m_ln_m,
                                   ptr(self.h_ll), ptr(self.h_mdl)))

    def describe(self):
        return arm_config("cfg3", self.w, self.units * self.world)

    def run_info(self):
        return {"distinct_subsets": self.fs.nsub, "parallelism": self.parallelism,
                "family_logical_bytes": self.family_bytes,
                "method": "LL(X|Pa) = sum n ln n over joint(X u Pa) - over joint(Pa)"}

    def cpu_baseline(self, budget, threads):
        def cols_fn(vs, nrows):
            return np.vstack([self.gdb.download(v, 0, nrows) for v in vs])

        qs = [(t, *ps) for t, ps in self.fs.families]
        return cpu_rate_queries(self.w, qs, budget, threads, cols_fn=cols_fn)


# kind::i8 tcgen05.mma throughput measured with tools/microbench6.cu on this pool's B200
# (A from TMEM, N >= 64): 8190 MAC/clk/SM; MEASURED_PEAKS.json has no int8 figure.
I8_MAC_PER_CLK_SM = 8190


class ItemsetRunner:
    """cfg4: supports of all 2- and 3-itemsets of the top-200 items.  The library picks the
    class (selector K4d on this sparse data; the tcgen05 bit-GEMM K4c for dense data); the
    kernel time is bracketed by the library's events around that class's launches."""

    kernel = "k_sel_gram"

    def __init__(self, args, world, rank, local, torch, ctx):
        from paper_1804_04640_b200 import workloads as W

        self.torch, self.ctx, self.world, self.rank = torch, ctx, world, rank
        self.config = "cfg4"
        m = args.m or 10_000_000
        self.w = W.cfg4(m=m)
        w = self.w
        t0 = time.perf_counter()
        self.gdb = w.build_device(ctx)
        sup = self.gdb.count_points([((v,), (1,)) for v in range(w.n)])
        self.sup = sup
        self.items = W.select_top_items(sup, w.meta["top"])
        self.gdb.bitmap_build(self.items)
        ctx.sync()
        self.build_s = time.perf_counter() - t0
        k = len(self.items)
        self.npairs = k * (k - 1) // 2
        self.ntri = k * (k - 1) * (k - 2) // 6
        self.units = self.npairs + self.ntri
        words = (m + 31) // 32
        self.algo_bytes = float(self.npairs * 2 + self.ntri * 3) * words * 4
        dev = "cuda"
        self.pairs = torch.empty((k, k), dtype=torch.int64, device=dev)
        self.triples = torch.empty(self.ntri, dtype=torch.int64, device=dev)
        self.h_pairs = torch.empty((k, k), dtype=torch.int64, pin_memory=True)
        self.h_triples = torch.empty(self.ntri, dtype=torch.int64, pin_memory=True)
        self.h2d = 4 * k
        self.d2h = 8 * (k * k + self.ntri)
        self.scaling = "weak"
        self.parallelism = "replica" if world == 1 else f"replicas x{world}"

    def roofline(self, k_ms, clocks):
        if self.ctx.itemset_class() == "selector":
            return self.roofline_selector(k_ms, clocks)
        return self.roofline_tensor(k_ms, clocks)

    def roofline_selector(self, k_ms, clocks):
        """K4d (rarest-item selection).  HBM roofline over its algorithmic bytes: k_sel_rowmask
        reads the k state-1 planes and writes the record-major rank masks (wr words per record);
        k_sel_gram reads each selector's plane and, per record holding the selector of rank r,
        the ceil(r/32) mask words below r.  Its issue bound is POPC: one per (8 x 4 Gram block, 32-record
        batch) counter, reported against 16 POPC/clk/SM (tools/microbench.cu)."""
        k, m = len(self.items), self.w.m
        words = -(-(-(-m // 32)) // 32) * 32  # plane words, padded to 32
        wr = 1 if k <= 32 else 2 if k <= 64 else 4 if k <= 128 else 8
        supp = sorted((int(self.sup[v]) for v in self.items), reverse=True)
        gather = sum(s * 4 * ((r + 31) // 32) for r, s in enumerate(supp) if r)
        algo = 4.0 * words * k + 4.0 * words * 32 * wr + 4.0 * words * (k - 1) + gather
        popc = 0.0
        for r, s in enumerate(supp):
            if r:
                nby, nbz = (r + 7) // 8, (r + 3) // 4
                nblk = sum(nbz - 2 * y for y in range(nby) if 2 * y < nbz)
                popc += -(-s // 32) * nblk * 32
        peak, src = load_peaks()
        achieved = algo / (k_ms / 1e3) / 1e9
        mhz = (clocks or {}).get("sm_mhz") or 1965.0
        popc_peak = 16.0 * 148 * mhz * 1e6
        return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": load_traffic("cfg4_selector"), "kernel": "k_sel_rowmask+k_sel_gram",
                "kernel_ms": k_ms, "algorithmic_bytes": algo, "peak_source": src,
                "popc": {"ops": popc, "achieved_per_s": popc / (k_ms / 1e3), "peak_per_s": popc_peak,
                         "frac": popc / (k_ms / 1e3) / popc_peak,
                         "note": "lower bound on issued POPC (batches assumed full)"},
                "logical_bytes": self.algo_bytes,
                "note": "selector class (DESIGN.md K4d): every itemset counted under its rarest item over "
                        "only the records holding it; logical_bytes = the per-itemset plane bytes of survey 8(d)"}

    def roofline_tensor(self, k_ms, clocks):
        """Tensor-bound: useful u8 x u8 MACs = (pairs + triples) x m, as int8 ops (2 per MAC),
        against the measured kind::i8 MMA rate at the sampled SM clock.  `computed_macs` adds
        the tiles' padding (rows x 16-column-rounded widths; K4c)."""
        k, m = len(self.items), self.w.m
        useful = float(self.npairs + self.ntri) * m
        rows = [b for b in range(k) for _ in range(b + 1)]  # (b, b) then (a, b) for a < b
        cols = 0
        for r0 in range(0, len(rows), 128):
            c0 = rows[r0] + 1
            while c0 < k:
                cols += min(256, (k - c0 + 15) // 16 * 16)
                c0 += 256
        computed = 128.0 * cols * ((m + 1023) // 1024 * 1024)
        mhz = (clocks or {}).get("sm_mhz") or 1965.0
        peak = 2.0 * I8_MAC_PER_CLK_SM * 148 * mhz * 1e6 / 1e12
        achieved = 2.0 * useful / (k_ms / 1e3) / 1e12
        return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TOP/s (int8)",
                "frac": achieved / peak, "traffic": load_traffic(self.config), "kernel": "k_itemsets_tc",
                "kernel_ms": k_ms, "useful_macs": useful, "computed_macs": computed,
                "computed_frac": 2.0 * computed / (k_ms / 1e3) / 1e12 / peak,
                "peak_source": f"measured: tools/microbench6.cu kind::i8 {I8_MAC_PER_CLK_SM} MAC/clk/SM x 148 SMs "
                               f"x {mhz:.0f} MHz (sampled clock)",
                "note": "kernel_ms spans k_pmt_transpose + the k_itemsets_tc launches (library events)"}

    def step(self):
        self.gdb.itemset_supports(self.items, self.pairs, self.triples)

    def e2e_step(self):
        self.gdb.itemset_supports(self.items, self.h_pairs, self.h_triples)

    def describe(self):
        return arm_config("cfg4", self.w, self.units * self.world)

    def run_info(self):
        return {"top": len(self.items), "parallelism": self.parallelism,
                "zipf_c": round(self.w.meta["zipf_c"], 6)}

    def cpu_baseline(self, budget, threads):
        """bitmap_count restatement on planes of the same items (downloaded columns), sampled."""
        import itertools

        O = _oracle()
        rows = min(self.w.m, 2_000_000)
        cols = {v: self.gdb.download(v, 0, rows) for v in self.items}
        planes = {(v, 1): O.bitmap_planes(cols[v], 1) for v in self.items}
        its = list(itertools.combinations(self.items, 3))
        probe = [tuple((v, 1) for v in t) for t in its[:2000]]
        t0 = time.perf_counter()
        O.bitmap_counts(planes, probe, rows, nthreads=threads)
        rate = len(probe) / (time.perf_counter() - t0)
        n = int(min(len(its), max(len(probe), rate * budget)))
        sample = [tuple((v, 1) for v in t) for t in its[:: max(1, len(its) // n)][:n]]
        t0 = time.perf_counter()
        O.bitmap_counts(planes, sample, rows, nthreads=threads)
        dt = time.perf_counter() - t0
        scale = rows / self.w.m
        return (len(sample) / dt * scale,
                f"{len(sample)} 3-itemsets on the first {rows} rows in {dt:.1f} s (bitmap_count restatement "
                f"oracle_bitmap_counts, {threads} threads; rate scaled x{scale:g} to m={self.w.m})")


# ---------------------------------------------------------------------------------------------
# per-query drop-in latency (reference harness.py:222-275: bench_random times Strategy.query
# one call at a time)


def _per_query_us(strategy, queries, make_agg, reps=1):
    for q in queries[:50]:  # warm-up (compiles / allocates outside the timed calls)
        strategy.query(q, make_agg(q))
    dts = []
    for _ in range(reps):
        for q in queries:
            agg = make_agg(q)
            t0 = time.perf_counter()
            strategy.query(q, agg)
            dts.append((time.perf_counter() - t0) * 1e6)
            agg.result()
    a = np.asarray(dts)
    return {"mean_us": float(a.mean()), "p50_us": float(np.median(a)), "p99_us": float(np.percentile(a, 99)),
            "queries_per_s": 1e6 / float(a.mean()), "calls": len(dts)}


def dropin_ours() -> dict:
    """cfg1's 1,000 queries, one GpuStrategy.query call each (built by make_strategies, the
    reference's registry API), with the aggregators the reference's own benchmark and scorers use."""
    import paper_1804_04640_b200 as cs
    from paper_1804_04640_b200 import workloads as W

    w = W.cfg1()
    built, _ = cs.make_strategies(w.host_db, ("gpu",))
    s = built["gpu"]
    qs = [cs.QuerySpec(q[0], tuple(q[1:])) for q in w.queries]
    out = {"workload": "cfg1 (n=20, m=1e4, 1,000 queries of target + 2 parents)",
           "strategy": "gpu (GpuStrategy.query, one call per query)",
           "NullSink": _per_query_us(s, qs, lambda q: cs.NullSink()),
           "LogLikelihood": _per_query_us(s, qs, lambda q: cs.LogLikelihood()),
           "RecordCollector": _per_query_us(s, qs, lambda q: cs.RecordCollector())}
    return out


def dropin_reference() -> dict:
    """The same calls through the reference's own strategies (baseline/_ref, one core)."""
    import tempfile

    ref = ROOT / "baseline" / "_ref"
    if not (ref / "countstream").exists():
        return {"unavailable": "baseline/_ref not installed"}
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_ref_"))
    sys.path.insert(0, str(ref))
    try:
        import countstream as R
    finally:
        sys.path.remove(str(ref))
    from paper_1804_04640_b200 import workloads as W

    w = W.cfg1()
    db = R.Database(w.host_db.data, [int(a) for a in w.arities])
    built, _ = R.make_strategies(db, ("bitmap", "radix"))
    qs = [R.QuerySpec(q[0], tuple(q[1:])) for q in w.queries]
    out = {"workload": "cfg1 (n=20, m=1e4, 1,000 queries of target + 2 parents)"}
    for name in ("bitmap", "radix"):
        out[name] = {"NullSink": _per_query_us(built[name], qs, lambda q: R.NullSink()),
                     "LogLikelihood": _per_query_us(built[name], qs, lambda q: R.LogLikelihood()),
                     "RecordCollector": _per_query_us(built[name], qs, lambda q: R.RecordCollector())}
    return out


# ---------------------------------------------------------------------------------------------
# arms


_NB = {}  # forked numba workers read the reference database / strategy from here


def _numba_worker(chunk):
    R, strat, db, cfg = _NB["R"], _NB["strat"], _NB["db"], _NB["cfg"]
    t0 = time.perf_counter()
    for q in chunk:
        qs = R.QuerySpec(q[0], tuple(q[1:]))
        agg = (R.LogLikelihood() if cfg in ("cfg1", "cfg5") else R.MdlScore.for_query(db, qs) if cfg == "cfg3"
               else R.NullSink())
        strat.query(qs, agg)
        agg.result()
    return time.perf_counter() - t0


def numba_reference(config, w, queries, budget_s, procs):
    """The reference itself: countstream's "radix" strategy (RadixStrategy, numba radix.py:33-156
    via harness.py:78-90, built by make_strategies, harness.py:125-158) installed unmodified in
    baseline/_ref, driven through its public Strategy.query with the reference's aggregators (NullSink for tables-only cfg2, LogLikelihood
    for cfg1, MdlScore for cfg3).  The reference is single-core by construction (GIL, numba
    without nogil), so it runs as `procs` forked processes over round-robin query slices
    (survey 8(d)); rate = sample queries / wall time of the parallel section.  None of this
    package's code runs in the timed region (the database is built from twin columns first)."""
    import multiprocessing as mp
    import tempfile

    ref = ROOT / "baseline" / "_ref"
    if not (ref / "countstream").exists():
        return {"unavailable": "baseline/_ref not installed (pip install --target baseline/_ref)"}
    if config not in ("cfg1", "cfg2", "cfg3"):
        return {"unavailable": f"{config}: the reference's int32 (n, m) Database does not fit host RAM"}
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_ref_"))
    sys.path.insert(0, str(ref))
    try:
        import countstream as R
    except Exception as e:  # pragma: no cover - environment
        return {"unavailable": f"cannot import the reference: {e!r}"[:200]}
    finally:
        sys.path.remove(str(ref))
    db = R.Database(host_columns(w).astype(np.int32), [int(a) for a in w.arities])
    built, failures = R.make_strategies(db, ("radix",))  # the reference's public registry
    if "radix" not in built:  # pragma: no cover
        return {"unavailable": f"make_strategies failed: {failures}"}
    strat = built["radix"]
    build = strat.build_seconds
    _NB.update(R=R, strat=strat, db=db, cfg=config)
    probe = list(queries[:4])
    rate1 = len(probe) / max(_numba_worker(probe), 1e-6)  # also compiles before the fork
    out = {"strategy": "countstream.RadixStrategy (numba)", "build_seconds": round(build, 3)}
    n1 = int(max(4, min(len(queries), rate1 * budget_s * 0.3)))
    dt1 = _numba_worker(list(queries[:n1]))
    out["single_core"] = {"value": n1 / dt1, "cores": 1,
                          "sample": f"first {n1} queries of the batch in {dt1:.1f} s, one process"}
    n = int(max(procs, min(len(queries), rate1 * procs * budget_s)))
    sample = list(queries[:n])
    chunks = [sample[i::procs] for i in range(procs)]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        pool.map(_numba_worker, [[q] for q in sample[:procs]])  # workers up
        t0 = time.perf_counter()
        pool.map(_numba_worker, chunks, chunksize=1)
        dt = time.perf_counter() - t0
    out.update(value=n / dt, cores=procs,
               sample=f"first {n} queries of the batch in {dt:.1f} s, {procs} forked processes (round robin)")
    _NB.clear()
    return out


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path on the host cores, rank 0 only.

    Two CPU implementations are timed: the oracle's C restatement of radix_query
    (oracle/radix_oracle.c, all host threads and one) -- the reference is Python, so there is no
    oracle/_ref build -- and the reference itself (numba RadixStrategy from baseline/_ref, all
    cores as forked processes, and one).  `value` is the faster of the two all-core figures.  No part of this package's engine is loaded: libcountgpu.so maps on
    first use (paper_1804_04640_b200/_native.py), and this arm never calls it."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if args.config == "cfg4":
        print(json.dumps({"impl": "reference", "unavailable": "--impl reference covers the counting-query "
                                                              "configs (default cfg2)"}), flush=True)
        return
    w, queries = workload(args.config, 1, 0, args.nq)
    limit = 12_500_000 if w.m > 20_000_000 else None
    rates, descs = [], []
    for i in range(args.warmup + args.steps):
        rot = (i * 997) % max(len(queries), 1)
        qs = list(queries[rot:]) + list(queries[:rot])
        rate, desc = cpu_rate_queries(w, qs, args.ref_budget, threads, row_limit=limit)
        if i >= args.warmup:
            rates.append(rate)
            descs.append(desc)
    v = statistics.mean(rates)
    r1, d1 = cpu_rate_queries(w, queries, args.ref_budget / 2, 1, row_limit=limit)
    nb = numba_reference(args.config, w, queries, args.ref_budget, threads)
    units = len(queries)
    port = v
    kind = "port"
    if nb.get("value", 0.0) > v:  # report the faster of the two CPU implementations (conservative)
        v, kind = nb["value"], "reference"
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * units / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded; DESIGN.md Workloads)", "config": arm_config(args.config, w, units),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": descs[-1] if kind == "port" else nb["sample"],
                         "port": {"value": port, "cores": threads, "sample": descs[-1]},
                         "port_single_core": {"value": r1, "cores": 1, "sample": d1},
                         "reference_numba": nb,
                         "value_source": "the faster of the C port (all threads) and the numba reference "
                                         "(all cores)"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_engine_loaded": _engine_loaded(),
    }
    if args.config == "cfg2" and not args.no_dropin:
        line["dropin"] = dropin_reference()
        line["native_engine_loaded"] = _engine_loaded()
    print(json.dumps(line), flush=True)


def _engine_loaded() -> bool:
    try:
        return "libcountgpu" in Path("/proc/self/maps").read_text()
    except OSError:  # pragma: no cover
        return False


def run_ours(args, world, rank, local):
    import torch

    from paper_1804_04640_b200.engine import GpuContext

    torch.cuda.set_device(local)
    distributed = world > 1 or "RANK" in os.environ  # launched by torchrun (even with one rank)
    if distributed:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = GpuContext(local)
    stream = torch.cuda.Stream()  # non-default: CUDA events and the library share it
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    R = {"cfg4": ItemsetRunner, "cfg3": FamilyRunner}.get(args.config, QueryRunner)
    r = R(args, world, rank, local, torch, ctx)
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")

    for _ in range(args.warmup):
        r.step()
    torch.cuda.synchronize()
    if distributed:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    l0 = ctx.launches
    kernel_ms = []
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if os.environ.get("CS_BENCH_NOFLUSH") != "1":  # diagnostic only: the line then says so
                flush.fill_(i)  # evict the database from L2 before every timed step (untimed)
            starts[i].record(stream)
            r.step()
            ends[i].record(stream)
            kernel_ms.append(ctx.last_kernel_ms())  # dominant kernel alone (library events)
        torch.cuda.synchronize()
    launches = ctx.launches - l0
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    step_ms = float(np.mean(ms))
    k_ms = (float(np.mean(kernel_ms)) if kernel_ms and min(kernel_ms) > 0 and not getattr(r, "kernel_is_step", False)
            else step_ms)
    if distributed:
        t = torch.tensor([step_ms, k_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        step_ms, k_ms = (float(x) for x in t.tolist())

    e2e_ms = []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        if distributed:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        r.e2e_step()
        dt = (time.perf_counter() - t0) * 1e3
        if i >= args.warmup:
            e2e_ms.append(dt)
    e2e_step = float(np.mean(e2e_ms))
    if distributed:
        t = torch.tensor([e2e_step], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_step = float(t.item())

    sharded = getattr(r, "sharded", False)
    total = r.units if sharded else r.units * world
    value = total / (step_ms / 1e3)
    if hasattr(r, "roofline"):
        roof = r.roofline(k_ms, clk.summary())
    else:
        roof = counting_roofline(r, k_ms)
    cfg = r.describe()
    run = r.run_info()
    run["db_build_seconds"] = round(r.build_s, 3)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": r.scaling,
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded; DESIGN.md Workloads)",
        "config": cfg,
        "run": run,
        "scanned_gbs": r.algo_bytes * world / (step_ms / 1e3) / 1e9,
        "roofline": roof,
        "e2e": {"value": total / (e2e_step / 1e3), "unit": UNIT, "h2d_bytes_per_step": r.h2d,
                "d2h_bytes_per_step": r.d2h, "ms_per_step": e2e_step},
        "gpu_launches": launches,
        "diag": {"step_ms": [round(x, 4) for x in ms[:8]]},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and args.config == "cfg2" and not args.no_dropin:
        line["dropin"] = dropin_ours()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, desc = r.cpu_baseline(args.ref_budget, threads)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc}
        if threads > 1:
            r1, d1 = r.cpu_baseline(args.ref_budget / 3, 1)
            line["cpu_baseline"]["single_core"] = {"value": r1, "cores": 1, "sample": d1}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if distributed:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nq", type=int, default=None, help="queries per GPU per step (default: the config's)")
    ap.add_argument("--m", type=int, default=None, help="rows (cfg4 only; default 1e7)")
    ap.add_argument("--ref-budget", type=float, default=12.0, help="seconds of CPU work per sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true", help="skip the per-query drop-in latency block")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        args.ref_budget = min(args.ref_budget, 6.0)
        run_reference(args, world, rank)
        return
    args.warmup = max(args.warmup, 3)
    run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
