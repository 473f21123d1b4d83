"""Python handles over the C ABI: device context, device database, query plans.

This is the layer the drop-in :class:`~paper_1804_04640_b200.harness.GpuStrategy`
and the batched workload drivers call.  Arrays passed in may be numpy (host)
or torch CUDA tensors (device); outputs land wherever the caller's array lives.
"""

from __future__ import annotations

import ctypes
import math
from ctypes import byref, c_int32, c_int64, c_void_p
from typing import Iterable, Sequence

import numpy as np

from . import _native as N
from ._native import check, lib, ptr

__all__ = ["GpuContext", "GpuDatabase", "QueryPlan", "FamilyScorer", "encode_queries"]


def encode_queries(queries: Iterable[Sequence[int]]) -> tuple[np.ndarray, np.ndarray]:
    """Variable tuples (target first) -> (var_off int32[nq+1], vars int32[sum k])."""
    qs = [tuple(int(v) for v in q) for q in queries]
    off = np.zeros(len(qs) + 1, dtype=np.int32)
    if qs:
        off[1:] = np.cumsum([len(q) for q in qs])
    flat = np.fromiter((v for q in qs for v in q), dtype=np.int32, count=int(off[-1]))
    return off, flat


def _load_message(source: str, buf, info: np.ndarray, arities) -> str:
    """The reference's DatabaseLoadError text (database.py:184-207, :53-77) for a
    cs_db_load_text failure; only the one offending line is read back on the host."""
    kind = int(info[0])
    if kind == N.CS_LOAD_NO_RECORDS:
        return f"{source}: no records found"
    if kind == N.CS_LOAD_NEGATIVE:
        return f"{source}: negative state {int(info[4])}; states must be >= 0"
    if kind == N.CS_LOAD_ARITY_COUNT:
        return f"expected {int(info[1])} arities, got {(int(info[4]),)}"
    if kind == N.CS_LOAD_ARITY_SHORT:
        var = int(info[5])
        return (f"row {int(info[4]) + 1}: variable {var} has state {int(info[6])}, "
                f"exceeding declared arity {int(arities[var])}")
    if kind == N.CS_LOAD_ARITY_ZERO:
        return "every arity must be at least 1"
    if kind == N.CS_LOAD_BAD_RECORD:
        rec, a, b = int(info[4]), int(info[5]), int(info[6])
        raw = bytes(buf[a:b].cpu().numpy() if hasattr(buf, "cpu") else buf[a:b])
        line = raw.decode("utf-8", errors="replace")
        kd, width = int(info[3]), int(info[1])
        toks = line.split() if kd < 0 else [t.strip() for t in line.split(chr(kd))]
        if len(toks) != width:
            return f"{source}: row {rec + 1}: expected {width} values, found {len(toks)}"
        for tok in toks:
            try:
                int(tok)
            except ValueError:
                return f"{source}: row {rec + 1}: non-integer token {tok!r}"
        return f"{source}: row {rec + 1}: token outside the device loader's ASCII integer grammar"
    return N.last_error()


class GpuContext:
    """One device + one stream (cs_ctx)."""

    def __init__(self, device: int = 0):
        h = c_void_p()
        check(lib.cs_ctx_create(int(device), byref(h)))
        self._h = h
        self.device = int(device)

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream: int | None) -> None:
        """Use an external cudaStream_t (e.g. ``torch.cuda.current_stream().cuda_stream``)."""
        check(lib.cs_ctx_set_stream(self._h, c_void_p(stream) if stream else None))

    def sync(self) -> None:
        check(lib.cs_ctx_sync(self._h))

    @property
    def launches(self) -> int:
        v = c_int64(0)
        check(lib.cs_ctx_launch_count(self._h, byref(v)))
        return int(v.value)

    def last_kernel_ms(self) -> float:
        """Device time of the last K1 (k_hist) launch, CUDA events on the context stream."""
        v = ctypes.c_float(0)
        check(lib.cs_ctx_last_kernel_ms(self._h, byref(v)))
        return float(v.value)

    def itemset_class(self) -> str:
        """Which class answered the last itemset_supports call: 'bitgemm', 'tensor', 'selector'."""
        v = c_int32(0)
        check(lib.cs_ctx_itemset_class(self._h, byref(v)))
        return {0: "none", 1: "bitgemm", 2: "tensor", 3: "selector"}[int(v.value)]

    # -- instance-shard merge through the C ABI (NCCL opened by the library) ------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        """A fresh 128-byte NCCL unique id (create on one rank, send to the others)."""
        buf = ctypes.create_string_buffer(128)
        check(lib.cs_comm_unique_id(buf))
        return buf.raw

    def comm_init(self, uid: bytes, rank: int, nranks: int) -> None:
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        check(lib.cs_comm_init(self._h, buf, int(rank), int(nranks)))

    def comm_destroy(self) -> None:
        check(lib.cs_comm_destroy(self._h))

    def reduce_tables(self, tables, op: int = 0, out=None, cells: int | None = None) -> None:
        """Sum device uint32/int32 tables over the communicator (cs_reduce_tables)."""
        n = int(tables.numel()) if cells is None else int(cells)
        check(lib.cs_reduce_tables(self._h, ptr(tables), n, int(op), ptr(out)))

    def all_gather(self, send, recv) -> None:
        """recv (device) = every rank's send (device) concatenated in rank order."""
        check(lib.cs_comm_all_gather(self._h, ptr(send), int(send.numel() * send.element_size()), ptr(recv)))

    def info(self) -> dict:
        a, b, c = c_int32(), c_int32(), c_int32()
        check(lib.cs_ctx_info(self._h, byref(a), byref(b), byref(c)))
        return {"num_sms": a.value, "hist_smem_bytes": b.value, "hist_ctas": c.value}

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.cs_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass


class GpuDatabase:
    """Device-resident uint8 column store (cs_db), one instance shard."""

    def __init__(self, ctx: GpuContext, handle, n: int, m: int, arities):
        self.ctx = ctx
        self._h = handle
        self.n = int(n)
        self.m = int(m)
        self.arities = np.asarray(arities, dtype=np.int64)
        self.arities.setflags(write=False)
        self.m_total = self.m

    @classmethod
    def from_columns(cls, ctx: GpuContext, cols, arities) -> "GpuDatabase":
        """cols: (n, m) uint8, numpy or torch CUDA tensor, rows = variables."""
        if hasattr(cols, "data_ptr"):
            n, m = cols.shape
            ld = cols.stride(0)
            src = cols
        else:
            cols = np.ascontiguousarray(cols, dtype=np.uint8)
            n, m = cols.shape
            ld = m
            src = cols
        ar = np.ascontiguousarray(arities, dtype=np.int32)
        h = c_void_p()
        check(lib.cs_db_create(ctx.handle, ptr(src), int(n), int(m), int(ld), ptr(ar), byref(h)))
        return cls(ctx, h, n, m, ar)

    @classmethod
    def from_text(cls, ctx: GpuContext, data, delimiter: str | None = None, arities=None,
                  source: str = "<text>") -> "GpuDatabase":
        """Parse delimited integer records on the device (cs_db_load_text; reference
        ``load_csv``, database.py:160-207, same grammar, 1-based shift, errors and messages).

        ``data``: bytes / uint8 numpy array (host) or a uint8 torch CUDA tensor.
        ``delimiter``: None sniffs ',' from the first record, else one character.
        """
        from .database import DatabaseLoadError, UnsupportedQueryError

        if isinstance(data, (bytes, bytearray, memoryview)):
            buf = np.frombuffer(data, dtype=np.uint8)
        else:
            buf = data
        nbytes = int(buf.numel() if hasattr(buf, "numel") else buf.size)
        if delimiter is None:
            delim = N.CS_DELIM_SNIFF
        else:
            raw = delimiter.encode()
            if len(raw) != 1:
                raise UnsupportedQueryError(
                    f"the device loader splits on one single-byte delimiter, got {delimiter!r}")
            delim = raw[0]
        ar = None if arities is None else np.ascontiguousarray(list(arities), dtype=np.int32)
        info = np.zeros(8, dtype=np.int64)
        h = c_void_p()
        rc = lib.cs_db_load_text(ctx.handle, ptr(buf) if nbytes else None, nbytes, int(delim),
                                 ptr(ar) if ar is not None and len(ar) else None,
                                 0 if ar is None else len(ar), byref(h), ptr(info))
        if rc == N.CS_ERR_PARSE:
            raise DatabaseLoadError(_load_message(source, buf, info, ar))
        check(rc)
        width = int(info[1])
        out_ar = np.empty(width, dtype=np.int32)
        check(lib.cs_db_arities(h, ptr(out_ar)))
        db = cls(ctx, h, width, int(info[2]), out_ar)
        db.load_info = {"delimiter": None if info[3] < 0 else chr(int(info[3])), "one_based": bool(info[7])}
        return db

    @classmethod
    def empty(cls, ctx: GpuContext, n: int, m: int, arities) -> "GpuDatabase":
        ar = np.ascontiguousarray(arities, dtype=np.int32)
        h = c_void_p()
        check(lib.cs_db_create_empty(ctx.handle, int(n), int(m), ptr(ar), byref(h)))
        return cls(ctx, h, n, m, ar)

    @property
    def handle(self):
        return self._h

    def generate(self, var: int, seed: int, thresholds, parents: Sequence[int] = (), row_offset: int = 0):
        thr = np.ascontiguousarray(thresholds, dtype=np.uint32).ravel()
        par = np.ascontiguousarray(list(parents), dtype=np.int32)
        check(
            lib.cs_db_generate(
                self._h, int(var), int(seed) & (2**64 - 1), int(row_offset), len(par),
                ptr(par) if len(par) else None, ptr(thr) if len(thr) else None, len(thr),
            )
        )

    def set_total_rows(self, m_total: int) -> None:
        check(lib.cs_db_set_total_rows(self._h, int(m_total)))
        self.m_total = int(m_total)

    def download(self, var: int, row0: int = 0, nrows: int | None = None) -> np.ndarray:
        nrows = self.m - row0 if nrows is None else nrows
        out = np.empty(nrows, dtype=np.uint8)
        check(lib.cs_db_download(self._h, int(var), int(row0), int(nrows), ptr(out)))
        return out

    def columns_ptr(self) -> tuple[int, int]:
        p = c_void_p()
        ld = c_int64()
        check(lib.cs_db_columns(self._h, byref(p), byref(ld)))
        return int(p.value or 0), int(ld.value)

    def bitmap_build(self, variables: Sequence[int] | None = None) -> None:
        if variables is None:
            check(lib.cs_bitmap_build(self._h, -1, None))
        else:
            vs = np.ascontiguousarray(list(variables), dtype=np.int32)
            check(lib.cs_bitmap_build(self._h, len(vs), ptr(vs) if len(vs) else None))

    def bitmap_plane(self, var: int, state: int) -> tuple[int, int]:
        p = c_void_p()
        w = c_int64()
        check(lib.cs_bitmap_plane(self._h, int(var), int(state), byref(p), byref(w)))
        return int(p.value or 0), int(w.value)

    def plan(self, queries, flags: int = 0) -> "QueryPlan":
        return QueryPlan(self, queries, flags)

    def query_batch(self, var_off: np.ndarray, vars_: np.ndarray, flags: int = 0, tables=None,
                    loglik=None, mi=None, nnz=None) -> None:
        """One-shot cs_query_batch (plan + execute + free) with caller-owned outputs."""
        check(lib.cs_query_batch(self._h, len(var_off) - 1, ptr(var_off), ptr(vars_), int(flags),
                                 ptr(tables), ptr(loglik), ptr(mi), ptr(nnz)))

    def query_one(self, vars_: np.ndarray, flags: int = 0, tables=None, loglik=None, mi=None, nnz=None) -> None:
        """One query (int32 variables, target first) through cs_query_one (latency class)."""
        check(lib.cs_query_one(self._h, len(vars_), ptr(vars_), int(flags), ptr(tables), ptr(loglik), ptr(mi),
                               ptr(nnz)))

    def count_points(self, assignments) -> np.ndarray:
        """assignments: iterable of (variables, states) pairs -> int64 counts."""
        assignments = list(assignments)
        off = np.zeros(len(assignments) + 1, dtype=np.int32)
        vs, ss = [], []
        for i, (v, s) in enumerate(assignments):
            vs.extend(int(x) for x in v)
            ss.extend(int(x) for x in s)
            off[i + 1] = len(vs)
        va = np.asarray(vs, dtype=np.int32)
        sa = np.asarray(ss, dtype=np.int32)
        out = np.zeros(len(assignments), dtype=np.int64)
        if len(assignments):
            check(
                lib.cs_count_points(
                    self._h, len(assignments), ptr(off), ptr(va) if len(va) else ptr(np.zeros(1, np.int32)),
                    ptr(sa) if len(sa) else ptr(np.zeros(1, np.int32)), ptr(out),
                )
            )
        return out

    def itemset_supports(self, items: Sequence[int], pairs: bool = True, triples: bool = True):
        """Supports of every 2- and 3-subset of ``items`` in state 1 (planes must exist).

        Returns (pairs (k, k) int64 with [a, b] filled for a < b, triples int64 in
        itertools.combinations order).  Outputs may also be given as device tensors.
        """
        it = np.ascontiguousarray(list(items), dtype=np.int32)
        k = len(it)
        pr = (np.zeros((k, k), dtype=np.int64) if pairs is True else pairs) if pairs is not False else None
        ntri = k * (k - 1) * (k - 2) // 6
        tr = (np.zeros(ntri, dtype=np.int64) if triples is True else triples) if triples is not False else None
        check(lib.cs_itemset_supports(self._h, k, ptr(it), ptr(pr), ptr(tr)))
        return pr, tr

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.cs_db_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class QueryPlan:
    """An uploaded batch of counting queries (cs_plan).

    ``queries`` are variable tuples, target first then parents.  Tables are
    packed: query q's cells are ``tables[table_off[q] : table_off[q] + cells[q]]``.
    """

    def __init__(self, db: GpuDatabase, queries, flags: int = 0):
        self.db = db
        if isinstance(queries, tuple) and len(queries) == 2 and isinstance(queries[0], np.ndarray):
            off, flat = queries
        else:
            off, flat = encode_queries(queries)
        self.var_off = np.ascontiguousarray(off, dtype=np.int32)
        self.vars = np.ascontiguousarray(flat, dtype=np.int32)
        self.nq = len(self.var_off) - 1
        self.flags = int(flags)
        h = c_void_p()
        vp = ptr(self.vars) if len(self.vars) else ptr(np.zeros(1, np.int32))
        check(lib.cs_plan_create(db.handle, self.nq, ptr(self.var_off), vp, self.flags, byref(h)))
        self._h = h
        self.cells = np.zeros(self.nq, dtype=np.int64)
        self.table_off = np.zeros(self.nq, dtype=np.int64)
        tot = c_int64()
        check(lib.cs_plan_info(h, ptr(self.cells), ptr(self.table_off), byref(tot)))
        self.total_cells = int(tot.value)
        self.r_target = db.arities[self.vars[self.var_off[:-1]]] if self.nq else np.zeros(0, np.int64)

    def execute(self, tables=None, loglik=None, mi=None, nnz=None) -> None:
        check(lib.cs_plan_execute(self._h, ptr(tables), ptr(loglik), ptr(mi), ptr(nnz)))

    def score(self, tables, loglik=None, mi=None, nnz=None) -> None:
        check(lib.cs_plan_score(self._h, ptr(tables), ptr(loglik), ptr(mi), ptr(nnz)))

    def compact(self, tables, nnz: np.ndarray):
        """Non-zero cells per query: (offsets[nq+1], cell_idx, n_ijk, n_ij) int64 host arrays."""
        nnz = np.asarray(nnz, dtype=np.int64)
        off = np.zeros(self.nq + 1, dtype=np.int64)
        off[1:] = np.cumsum(nnz)
        tot = int(off[-1])
        ci = np.empty(max(tot, 1), dtype=np.int64)
        a = np.empty(max(tot, 1), dtype=np.int64)
        b = np.empty(max(tot, 1), dtype=np.int64)
        if tot:
            check(lib.cs_plan_compact(self._h, ptr(tables), ptr(off[:-1].copy()), tot, ptr(ci), ptr(a), ptr(b)))
        return off, ci[:tot], a[:tot], b[:tot]

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.cs_plan_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class FamilyScorer:
    """LL and MDL of many (target, parents) families from one histogram launch.

    LL(X | Pa) = sum_cells n ln n over joint(X u Pa) - sum_cells n ln n over joint(Pa), so a
    batch of families needs only its *distinct variable subsets* counted (for every parent set
    of size <= 3 over n=37 variables: 74,518 subsets for 288,859 families).  The subset sums
    come from a CS_NLOGN plan; cs_family_scores combines them and adds the MDL penalty
    0.5 ln(m) (r_i - 1) q_i (aggregators.py:191-193).
    """

    def __init__(self, db: GpuDatabase, families, m_total: int | None = None):
        self.db = db
        fams = [(int(t), tuple(int(p) for p in ps)) for t, ps in families]
        index: dict = {}
        s_idx = np.empty(len(fams), dtype=np.int32)
        p_idx = np.empty(len(fams), dtype=np.int32)
        pen = np.empty(len(fams), dtype=np.float64)
        m = int(m_total if m_total is not None else db.m_total)
        lnm = math.log(m)
        ar = db.arities
        for f, (t, ps) in enumerate(fams):
            key = tuple(sorted((t,) + ps))
            s_idx[f] = index.setdefault(key, len(index))
            if ps:
                pk = tuple(sorted(ps))
                p_idx[f] = index.setdefault(pk, len(index))
            else:
                p_idx[f] = -1
            q_i = 1
            for p in ps:
                q_i *= int(ar[p])
            pen[f] = 0.5 * lnm * (int(ar[t]) - 1) * q_i
        self.families = fams
        self.subsets = list(index)
        self.s_idx, self.p_idx, self.penalty = s_idx, p_idx, pen
        self.m_ln_m = m * lnm
        self.plan = QueryPlan(db, self.subsets, N.CS_NLOGN)
        self.nfam = len(fams)
        self.nsub = len(self.subsets)

    def to_device(self, torch):
        """Move the per-family index/penalty arrays to the device (bench: resident inputs)."""
        self.s_idx = torch.from_numpy(self.s_idx).cuda()
        self.p_idx = torch.from_numpy(self.p_idx).cuda()
        self.penalty = torch.from_numpy(self.penalty).cuda()
        return self

    def run(self, nlogn, ll=None, mdl=None) -> None:
        """nlogn: float64[nsub] work array (host or device); ll / mdl: float64[nfam] outputs."""
        self.plan.execute(loglik=nlogn)
        check(lib.cs_family_scores(self.db.ctx.handle, self.nfam, ptr(nlogn), self.nsub, ptr(self.s_idx),
                                   ptr(self.p_idx), ptr(self.penalty), self.m_ln_m, ptr(ll), ptr(mdl)))

    def scores(self) -> tuple[np.ndarray, np.ndarray]:
        nl = np.zeros(self.nsub)
        ll = np.zeros(self.nfam)
        mdl = np.zeros(self.nfam)
        self.run(nl, ll, mdl)
        return ll, mdl
