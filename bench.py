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
             are summed with an NCCL all-reduce, then LL + MI are scored (strong scaling).

value      units/s over all ranks, device-timed (CUDA events on the launch stream, max over
           ranks), database + plan resident in HBM; L2 flushed (256 MB write) before every
           timed step.
e2e        through the C ABI with HOST buffers each step: query descriptors in, tables /
           scores / supports out to pinned host memory.
roofline   the dominant kernel (k_hist, or k_itemsets for cfg4): algorithmic bytes per launch
            / its device time (library CUDA events, same stream).
cpu_baseline  the oracle's C restatement of the reference path (port, all host threads) on
           a bounded sample of the same workload.
--impl reference  times that CPU port alone (the reference itself is pure Python + numba
           and cannot travel to the GPU box).
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
        w = W.cfg5(nq=nq_override or 2_000)
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
        self.plan = QueryPlan(self.gdb, self.queries, flags)
        self.units = self.plan.nq
        if self.sharded:
            from paper_1804_04640_b200.parallel import PipelinedInstanceSharded

            self.pipe = PipelinedInstanceSharded(self.gdb, self.queries, nbatch=4)
        dev = "cuda"
        self.tables = (torch.empty(max(self.plan.total_cells, 1), dtype=torch.int32, device=dev)
                       if (self.want_tables or self.sharded) else None)
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
        self.parallelism = (f"instance-shard x{world} + NCCL all-reduce" if self.sharded
                            else f"query-shard x{world}")

    def step(self):
        if self.sharded:
            # four query slices: slice b's NCCL all-reduce (uint32 sum == int32 sum bitwise)
            # overlaps slice b+1's scan; each slice is scored after its merge
            self.pipe.run(loglik=self.ll, mi=self.mi)
        else:
            self.plan.execute(tables=self.tables, loglik=self.ll, mi=self.mi)

    def e2e_step(self):
        if self.sharded:
            self.step()
            self.h_ll.copy_(self.ll)
            self.h_mi.copy_(self.mi)
            self.torch.cuda.synchronize()
            return
        self.gdb.query_batch(self.off, self.flat, self.flags, tables=self.h_tables, loglik=self.h_ll,
                             mi=self.h_mi)

    def describe(self):
        return {"workload": self.w.name, "n": self.w.n, "m": self.w.m, "queries_per_step": self.units,
                "total_cells": int(self.plan.total_cells), "parallelism": self.parallelism,
                "outputs": "+".join(x for x, f in (("tables", self.want_tables), ("loglik", self.want_ll),
                                                    ("mi", self.want_mi)) if f)}

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
        return {"workload": "cfg3", "n": self.w.n, "m": self.w.m, "families_per_step": self.units,
                "distinct_subsets": self.fs.nsub, "parallelism": self.parallelism, "outputs": "loglik+mdl",
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
        return {"workload": "cfg4", "items": self.w.n, "m": self.w.m, "top": len(self.items),
                "itemsets_per_step": self.units, "parallelism": self.parallelism,
                "outputs": "pair+triple supports", "zipf_c": round(self.w.meta["zipf_c"], 6)}

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
# arms


def run_reference(args, world, rank):
    """--impl reference: the CPU port of the reference path, rank 0 only."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    if args.config == "cfg4":
        raise SystemExit("--impl reference supports the query configs (default cfg2)")
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
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * len(queries) / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": {"workload": w.name, "m": w.m, "n": w.n, "queries": len(queries)},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": descs[-1]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
            flush.fill_(i)  # evict the database from L2 before every timed step (untimed)
            starts[i].record(stream)
            r.step()
            ends[i].record(stream)
            kernel_ms.append(ctx.last_kernel_ms())  # dominant kernel alone (library events)
        torch.cuda.synchronize()
    launches = ctx.launches - l0
    ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    step_ms = float(np.mean(ms))
    k_ms = float(np.mean(kernel_ms)) if kernel_ms and min(kernel_ms) > 0 else step_ms
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
    peak, peak_src = load_peaks()
    achieved = r.algo_bytes / (k_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": load_traffic(r.config), "kernel": r.kernel,
            "kernel_ms": k_ms, "peak_source": peak_src,
            "note": "achieved = algorithmic bytes per launch / kernel time; frac > 1 means the "
                    "kernel reuses data from L2/SMEM across queries (reuse regime)"}
    if hasattr(r, "roofline"):
        roof = r.roofline(k_ms, clk.summary())
    cfg = r.describe()
    cfg.update({"l2": "flushed (256 MB write) before every timed step", "db_build_seconds": round(r.build_s, 3)})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": r.scaling,
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded; DESIGN.md Workloads)",
        "config": cfg,
        "scanned_gbs": r.algo_bytes * world / (step_ms / 1e3) / 1e9,
        "roofline": roof,
        "e2e": {"value": total / (e2e_step / 1e3), "unit": UNIT, "h2d_bytes_per_step": r.h2d,
                "d2h_bytes_per_step": r.d2h, "ms_per_step": e2e_step},
        "gpu_launches": launches,
        "diag": {"step_ms": [round(x, 4) for x in ms[:8]]},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, desc = r.cpu_baseline(args.ref_budget, threads)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "sample": desc}
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
