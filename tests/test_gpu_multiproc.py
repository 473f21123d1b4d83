"""Multi-process instance sharding with the REAL kernels: two
processes share the one GPU of the test box, each counting its row shard with libcountgpu
(CS_PARTIAL plans, generated with global row ids), merging over gloo on host copies (no
process waits on another's kernels), scoring the merged tables on the device; checked against
the oracle on the whole database.  Both merges: all-reduce + score everything, and
reduce-scatter ownership + per-owner scoring + all-gather of the scalars.  Plus the C-ABI NCCL
path (cs_comm_init / cs_reduce_tables) on a one-rank communicator."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen_twin
        import oracle as O
        import paper_1804_04640_b200 as cs
        from paper_1804_04640_b200 import parallel, workloads
        from paper_1804_04640_b200._native import CS_PARTIAL, CS_WANT_TABLES
        from paper_1804_04640_b200.engine import QueryPlan

        ctx = cs.shared_context(0)
        w = workloads.cfg5(nq=120, m=400_037, n=40, seed=11)
        r0, nr = parallel.shard_rows(w.m, world, rank)
        gdb = w.build_device(ctx, row_offset=r0, m_shard=nr)  # sets the global m
        # all-reduce: partial tables -> host -> gloo sum -> device score of every query
        plan = QueryPlan(gdb, w.queries, CS_PARTIAL | CS_WANT_TABLES)
        part = np.zeros(plan.total_cells, dtype=np.uint32)
        plan.execute(tables=part)
        t = torch.from_numpy(part.view(np.int32).copy())
        dist.all_reduce(t)
        merged = t.numpy().view(np.uint32)
        ll = np.zeros(plan.nq)
        mi = np.zeros(plan.nq)
        plan.score(merged, loglik=ll, mi=mi)
        # reduce-scatter ownership
        rs = parallel.ReduceScatterInstanceSharded(gdb, w.queries, world, rank, comm="host")
        ll_rs = torch.zeros(len(w.queries), dtype=torch.float64, device="cuda")
        mi_rs = torch.zeros_like(ll_rs)
        nnz_rs = torch.zeros(len(w.queries), dtype=torch.int64, device="cuda")
        rs.run(loglik=ll_rs, mi=mi_rs, nnz=nnz_rs)
        torch.cuda.synchronize()
        # oracle on the whole database
        cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
        u8 = np.vstack([cols[v] for v in range(w.n)])
        otabs, _, oll, omi, onnz = O.dense_tables(u8, w.arities, w.queries)
        res = {
            "tables": bool(np.array_equal(merged, otabs)),
            "ll": bool(np.allclose(ll, oll, rtol=1e-9, atol=1e-9)),
            "mi": bool(np.allclose(mi, omi, rtol=1e-9, atol=1e-12)),
            "rs_ll": bool(np.allclose(ll_rs.cpu().numpy(), oll, rtol=1e-9, atol=1e-9)),
            "rs_mi": bool(np.allclose(mi_rs.cpu().numpy(), omi, rtol=1e-9, atol=1e-12)),
            "rs_nnz": bool(np.array_equal(nnz_rs.cpu().numpy(), onnz)),
            "rows": nr,
        }
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_processes_real_kernels_gloo_merge():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for rank, r in res:
        assert r["rows"] > 0
        assert all(v for k, v in r.items() if k != "rows"), (rank, r)


def test_c_abi_nccl_single_rank():
    """cs_comm_unique_id / cs_comm_init / cs_reduce_tables on a one-rank communicator: the
    all-reduce is the identity, the reduce-scatter returns the whole buffer; and the
    reduce-scatter runner over the library communicator equals the fused scores."""
    import torch

    import paper_1804_04640_b200 as cs
    from paper_1804_04640_b200 import parallel, workloads
    from paper_1804_04640_b200._native import CS_REDUCE_ALLREDUCE, CS_REDUCE_SCATTER
    from paper_1804_04640_b200.engine import QueryPlan

    ctx = cs.shared_context(0)
    uid = ctx.comm_unique_id()
    assert len(uid) == 128
    ctx.comm_init(uid, 0, 1)
    try:
        x = torch.arange(1000, dtype=torch.int32, device="cuda")
        ctx.reduce_tables(x, CS_REDUCE_ALLREDUCE)
        out = torch.zeros_like(x)
        ctx.reduce_tables(x, CS_REDUCE_SCATTER, out)
        ctx.sync()
        assert torch.equal(x, torch.arange(1000, dtype=torch.int32, device="cuda"))
        assert torch.equal(out, x)
        w = workloads.cfg5(nq=80, m=200_001, n=30, seed=5)
        gdb = w.build_device(ctx)
        rs = parallel.ReduceScatterInstanceSharded(gdb, w.queries, 1, 0, comm="cs")
        ll = torch.zeros(len(w.queries), dtype=torch.float64, device="cuda")
        rs.run(loglik=ll)
        torch.cuda.synchronize()
        plan = QueryPlan(gdb, w.queries)
        ll0 = np.zeros(plan.nq)
        plan.execute(loglik=ll0)
        assert np.allclose(ll.cpu().numpy(), ll0, rtol=1e-12, atol=1e-9)
    finally:
        ctx.comm_destroy()
