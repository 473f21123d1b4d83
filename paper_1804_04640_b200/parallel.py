"""Multi-GPU partitioning of counting work (one process per GPU, torch.distributed / NCCL).

Two shardings:

* **instance sharding** -- counts are additive over disjoint row ranges: rank g holds rows
  ``shard_rows(m, N, g)``, counts partial uint32 tables (``CS_PARTIAL``), the tables are summed
  with one all-reduce (:func:`merge_tables_`) and scored with the global m; or, with
  :class:`ReduceScatterInstanceSharded`, reduce-scattered so each rank receives and scores only
  the queries it owns (half the NVLink volume of the all-reduce), then the fp64 scores are
  all-gathered;
* **query sharding** -- when the database fits on every GPU, each rank runs a cost-balanced
  slice of the batch (:func:`shard_queries`); no data-path collective.

The reference has no parallel code (survey section 2); these functions are the plumbing around
the C ABI.  They only use ``torch.distributed`` collectives, so the same code runs over NCCL on
GPUs and over gloo on CPU (tests/test_multirank.py).
"""

from __future__ import annotations

import heapq

import numpy as np

__all__ = ["shard_rows", "shard_queries", "merge_tables_", "gather_by_index", "InstanceShardedPlan",
           "PipelinedInstanceSharded", "owner_split", "ReduceScatterInstanceSharded"]


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """(first global row, row count) of rank's instance shard: contiguous, sizes differ by <= 1
    multiple of 256 rows (the column alignment)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    per = -(-m // world)
    per = -(-per // 256) * 256
    r0 = min(m, rank * per)
    return r0, max(0, min(per, m - r0))


def shard_queries(queries, world: int, rank: int, cost=None) -> tuple[list, np.ndarray]:
    """Longest-processing-time split of a query batch; returns (rank's queries, their indices).

    ``cost(q)`` defaults to the query's byte volume (number of variables), the k*m bytes a
    query streams.
    """
    qs = list(queries)
    cost = cost or (lambda q: len(q))
    order = sorted(range(len(qs)), key=lambda i: (-cost(qs[i]), i))
    heap = [(0.0, r) for r in range(world)]
    owner = np.empty(len(qs), dtype=np.int64)
    for i in order:
        load, r = heapq.heappop(heap)
        owner[i] = r
        heapq.heappush(heap, (load + cost(qs[i]), r))
    idx = np.nonzero(owner == rank)[0]
    return [qs[i] for i in idx], idx


def merge_tables_(tables, group=None):
    """In-place sum of partial uint32 tables across ranks (int32 view: bitwise identical sum)."""
    import torch
    import torch.distributed as dist

    t = tables if tables.dtype == torch.int32 else tables.view(torch.int32)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return tables


def gather_by_index(local_values, local_index, total: int, group=None):
    """Assemble per-query results computed on different ranks into one array (all ranks)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    vals = torch.as_tensor(np.asarray(local_values, dtype=np.float64))
    idx = torch.as_tensor(np.asarray(local_index, dtype=np.int64))
    n = torch.tensor([len(idx)], dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    mx = int(max(int(s) for s in sizes))
    pv = torch.zeros(mx, dtype=torch.float64)
    pi = torch.full((mx,), -1, dtype=torch.int64)
    pv[: len(idx)] = vals
    pi[: len(idx)] = idx
    gv = [torch.zeros(mx, dtype=torch.float64) for _ in range(world)]
    gi = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(gv, pv, group=group)
    dist.all_gather(gi, pi, group=group)
    out = np.zeros(total)
    for v, i in zip(gv, gi):
        keep = i >= 0
        out[i[keep].numpy()] = v[keep].numpy()
    return out


class InstanceShardedPlan:
    """One rank's share of an instance-sharded batch on the device.

    ``gdb`` holds this rank's rows (``build_device(ctx, row_offset, m_shard)``) and knows the
    global m (``set_total_rows``).  ``run()`` counts partial tables, all-reduces them over the
    process group (NCCL) and scores the merged tables with the fused fp64 epilogue.
    """

    def __init__(self, gdb, queries, torch_device="cuda", group=None, tables=None):
        import torch

        from . import _native as N
        from .engine import QueryPlan

        self.plan = QueryPlan(gdb, queries, N.CS_PARTIAL | N.CS_WANT_TABLES)
        n = max(self.plan.total_cells, 1)
        # `tables`: a caller-owned device buffer of >= total_cells words (shared by consecutive plans)
        self.tables = (tables[:n] if tables is not None and tables.numel() >= n
                       else torch.empty(n, dtype=torch.int32, device=torch_device))
        self.group = group

    def run(self, loglik=None, mi=None, nnz=None):
        self.plan.execute(tables=self.tables)
        merge_tables_(self.tables, self.group)
        self.plan.score(self.tables, loglik=loglik, mi=mi, nnz=nnz)
        return self.tables


class PipelinedInstanceSharded:
    """Instance-sharded batch in ``nbatch`` query slices whose merges overlap the next slice's
    scan (survey 8(e)): slice b's partial tables are all-reduced asynchronously (NCCL runs on
    its own stream after the compute stream's work so far) while slice b+1 is counted; slice
    b is scored once its merge is waited on.  Results are identical to
    :class:`InstanceShardedPlan` over the whole batch (counts are additive, scoring is per
    query).  As for every torch.distributed call here, the library context's stream must be
    torch's current stream (``ctx.set_stream(torch.cuda.current_stream().cuda_stream)`` under
    ``torch.cuda.stream(s)``), so the collectives are ordered after the kernels that feed them.
    """

    def __init__(self, gdb, queries, nbatch: int = 4, torch_device="cuda", group=None):
        import torch

        from . import _native as N
        from .engine import QueryPlan

        qs = list(queries)
        nbatch = max(1, min(nbatch, len(qs)))
        cuts = [len(qs) * i // nbatch for i in range(nbatch + 1)]
        self.slices = [(cuts[i], cuts[i + 1]) for i in range(nbatch) if cuts[i + 1] > cuts[i]]
        self.plans = [QueryPlan(gdb, qs[a:b], N.CS_PARTIAL | N.CS_WANT_TABLES) for a, b in self.slices]
        self.tables = [torch.empty(max(p.total_cells, 1), dtype=torch.int32, device=torch_device)
                       for p in self.plans]
        self.nq = len(qs)
        self.group = group

    def run(self, loglik=None, mi=None, nnz=None):
        """loglik / mi / nnz: device tensors over the whole batch (or None)."""
        import torch.distributed as dist

        def part(x, a, b):
            return None if x is None else x[a:b]

        pending = None
        for i, (plan, tab) in enumerate(zip(self.plans, self.tables)):
            plan.execute(tables=tab)
            work = dist.all_reduce(tab, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
            if pending is not None:
                j, w = pending
                w.wait()  # the compute stream waits for slice j's merge, after slice i's scan
                a, b = self.slices[j]
                self.plans[j].score(self.tables[j], loglik=part(loglik, a, b), mi=part(mi, a, b),
                                    nnz=part(nnz, a, b))
            pending = (i, work)
        j, w = pending
        w.wait()
        a, b = self.slices[j]
        self.plans[j].score(self.tables[j], loglik=part(loglik, a, b), mi=part(mi, a, b), nnz=part(nnz, a, b))


def owner_split(cells, world: int) -> list:
    """Owner rank of each query: longest-processing-time on table cells, so the owners' merged
    segments (and the reduce-scatter's equal-size slices) are balanced.  Returns, per rank, the
    ascending query indices it owns."""
    cells = [int(c) for c in cells]
    order = sorted(range(len(cells)), key=lambda i: (-cells[i], i))
    heap = [(0, r) for r in range(world)]
    owned = [[] for _ in range(world)]
    for i in order:
        load, r = heapq.heappop(heap)
        owned[r].append(i)
        heapq.heappush(heap, (load + cells[i], r))
    return [sorted(o) for o in owned]


class ReduceScatterInstanceSharded:
    """Instance sharding with per-owner scoring (survey 8(e): "NCCL ReduceScatter; each GPU owns
    about 1/N of the batch's queries (by table bytes), scores them, then gathers the scalars").

    Every rank counts its rows for every query, but through one plan per owner whose tables land
    in that owner's slice of a ``world x S`` buffer (S = the largest owner's cells; the padding
    stays zero).  One reduce-scatter leaves rank r exactly the merged tables of the queries it
    owns; it scores them with the global m and the fp64 scores are all-gathered.  NVLink volume:
    (N-1)/N of the tables instead of the all-reduce's 2(N-1)/N.

    ``comm``: ``"torch"`` -- torch.distributed (NCCL for CUDA tensors); ``"host"`` -- the same
    collectives on host copies (gloo process groups, tests); ``"cs"`` -- the library's own NCCL
    communicator (``GpuContext.comm_init``; the C ABI path for non-torch callers).
    """

    def __init__(self, gdb, queries, world: int, rank: int, comm: str = "torch", torch_device="cuda",
                 group=None, buf=None):
        import torch

        from . import _native as N
        from .engine import QueryPlan

        qs = [tuple(int(v) for v in q) for q in queries]
        ar = gdb.arities
        cells = [int(np.prod([int(ar[v]) for v in q], dtype=np.int64)) for q in qs]
        self.owned = owner_split(cells, world)
        self.world, self.rank, self.comm, self.group = world, rank, comm, group
        self.gdb = gdb
        self.nq = len(qs)
        self.plans = [QueryPlan(gdb, [qs[i] for i in o], N.CS_PARTIAL | N.CS_WANT_TABLES) if o else None
                      for o in self.owned]
        self.S = max(1, max((p.total_cells for p in self.plans if p is not None), default=1))
        self.S = -(-self.S // 64) * 64
        # `buf`: a caller-owned zeroed device buffer of >= world * S + S words, shared by
        # consecutive runners (the padding of every owner slice must read zero)
        if buf is not None and buf.numel() >= (world + 1) * self.S:
            self.buf, self.out = buf[: world * self.S], buf[world * self.S: (world + 1) * self.S]
        else:
            self.buf = torch.zeros(world * self.S, dtype=torch.int32, device=torch_device)
            self.out = torch.empty(self.S, dtype=torch.int32, device=torch_device)
        self.qmax = max(1, max(len(o) for o in self.owned))
        self.idx = torch.full((world, self.qmax), -1, dtype=torch.int64)
        for r, o in enumerate(self.owned):
            self.idx[r, : len(o)] = torch.as_tensor(o, dtype=torch.int64)
        self.idx = self.idx.to(torch_device)

    def _reduce_scatter(self):
        import torch
        import torch.distributed as dist

        if self.comm == "cs":
            from . import _native as N

            self.gdb.ctx.reduce_tables(self.buf, N.CS_REDUCE_SCATTER, self.out)
        elif self.comm == "host":
            torch.cuda.synchronize()
            hb, ho = self.buf.cpu(), torch.empty(self.S, dtype=torch.int32)
            dist.reduce_scatter_tensor(ho, hb, op=dist.ReduceOp.SUM, group=self.group)
            self.out.copy_(ho)
        else:
            dist.reduce_scatter_tensor(self.out, self.buf, op=dist.ReduceOp.SUM, group=self.group)

    def _all_gather(self, x):
        import torch
        import torch.distributed as dist

        full = torch.empty(self.world * self.qmax, dtype=x.dtype, device=x.device)
        if self.comm == "cs":
            self.gdb.ctx.all_gather(x, full)
            self.gdb.ctx.sync()
        elif self.comm == "host":
            torch.cuda.synchronize()
            hf = torch.empty(self.world * self.qmax, dtype=x.dtype)
            dist.all_gather_into_tensor(hf, x.cpu(), group=self.group)
            full.copy_(hf)
        else:
            dist.all_gather_into_tensor(full, x, group=self.group)
        return full

    def run(self, loglik=None, mi=None, nnz=None):
        """Count (every owner's plan over this rank's rows), reduce-scatter, score the owned
        queries, all-gather.  loglik / mi / nnz: device tensors over the whole batch (or None)."""
        import torch

        for r, p in enumerate(self.plans):
            if p is not None:
                sl = self.buf[r * self.S: (r + 1) * self.S]
                sl[p.total_cells:].zero_()  # a shared buffer's padding from an earlier runner
                p.execute(tables=sl[: p.total_cells])
        self._reduce_scatter()
        own = self.plans[self.rank]
        outs = {}
        for name, dst, dt in (("loglik", loglik, torch.float64), ("mi", mi, torch.float64), ("nnz", nnz, torch.int64)):
            if dst is None:
                continue
            outs[name] = (dst, torch.zeros(self.qmax, dtype=dt, device=self.buf.device))
        if own is not None and outs:
            n = own.nq
            own.score(self.out[: own.total_cells], **{k: v[1][:n] for k, v in outs.items()})
        self.gdb.ctx.sync()
        keep = self.idx.reshape(-1) >= 0
        for name, (dst, mine) in outs.items():
            full = self._all_gather(mine)
            dst[self.idx.reshape(-1)[keep]] = full[keep]
        return self.out
