"""Multi-process (gloo, world_size 2, CPU) coverage of the N>1 paths.

The instance-sharded merge algebra: per-rank partial tables over disjoint row shards, summed
with the same all-reduce helper the GPU path uses (merge_tables_), equal the full-database
tables; scores of the merged tables equal the full scores.  Query sharding: the LPT split
covers every query exactly once and the gathered results equal the unsharded ones.  The
oracle stands in for the per-rank device counts (no GPU here).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle as O
        from paper_1804_04640_b200 import parallel, workloads

        w = workloads.cfg2(nq=60, m=50_003, seed=9)
        import gen_twin

        cols = gen_twin.generate_workload_columns(w, np.arange(w.m))
        u8 = np.vstack([cols[v] for v in range(w.n)])
        # instance sharding: partial tables on this rank's rows
        r0, nr = parallel.shard_rows(w.m, world, rank)
        part, off, _, _ = O.radix_tables(np.ascontiguousarray(u8[:, r0:r0 + nr]), w.arities, w.queries)
        t = torch.from_numpy(part.view(np.int32).copy())
        parallel.merge_tables_(t)
        full, _, ll_full, _ = O.radix_tables(u8, w.arities, w.queries)
        ok_tables = bool(np.array_equal(t.numpy().view(np.uint32), full))
        # query sharding + gather
        mine, idx = parallel.shard_queries(w.queries, world, rank)
        _, _, ll_mine, _ = O.radix_tables(u8, w.arities, mine)
        got = parallel.gather_by_index(ll_mine, idx, len(w.queries))
        ok_gather = bool(np.allclose(got, ll_full, rtol=1e-12, atol=0))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([len(idx)], dtype=torch.int64))
        ok_cover = int(sum(int(s) for s in sizes)) == len(w.queries)
        # reduce-scatter ownership (parallel.ReduceScatterInstanceSharded's layout): every rank
        # lays its partial tables out per owner in a world x S buffer; one reduce-scatter leaves
        # each owner exactly the merged tables of its queries
        cells = [int(np.prod([int(w.arities[v]) for v in qq])) for qq in w.queries]
        owned = parallel.owner_split(cells, world)
        S = max(sum(cells[i] for i in o) for o in owned)
        buf = np.zeros(world * S, dtype=np.uint32)
        for r, o in enumerate(owned):
            pt, _, _, _ = O.radix_tables(np.ascontiguousarray(u8[:, r0:r0 + nr]), w.arities, [w.queries[i] for i in o])
            buf[r * S: r * S + len(pt)] = pt
        out = torch.zeros(S, dtype=torch.int32)
        dist.reduce_scatter_tensor(out, torch.from_numpy(buf.view(np.int32)))
        mine_full, _, mine_ll, _ = O.radix_tables(u8, w.arities, [w.queries[i] for i in owned[rank]])
        ok_rs = bool(np.array_equal(out.numpy().view(np.uint32)[: len(mine_full)], mine_full))
        ok_rs &= bool((out.numpy()[len(mine_full):] == 0).all())
        ok_cover &= sorted(i for o in owned for i in o) == list(range(len(w.queries)))
        ok_tables &= ok_rs
        q.put((rank, ok_tables, ok_gather, ok_cover, nr))
    finally:
        dist.destroy_process_group()


def test_shard_rows_cover_exactly():
    from paper_1804_04640_b200 import parallel

    for m in (1, 255, 256, 1000, 100_000_000):
        for world in (1, 2, 3, 8):
            got = [parallel.shard_rows(m, world, r) for r in range(world)]
            assert sum(n for _, n in got) == m
            pos = 0
            for r0, n in got:
                if n:
                    assert r0 == pos and r0 % 256 == 0
                pos += n


def test_shard_queries_balanced():
    from paper_1804_04640_b200 import parallel

    rng = np.random.default_rng(1)
    qs = [tuple(range(int(k))) for k in rng.integers(1, 7, size=1000)]
    loads, seen = [], []
    for r in range(4):
        mine, idx = parallel.shard_queries(qs, 4, r)
        loads.append(sum(len(q) for q in mine))
        seen.extend(idx.tolist())
    assert sorted(seen) == list(range(1000))
    assert max(loads) - min(loads) <= 6


def test_two_rank_gloo_merge_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_tables, ok_gather, ok_cover, nr in res:
        assert ok_tables, f"rank {rank}: merged partial tables differ from the full tables"
        assert ok_gather, f"rank {rank}: gathered query-shard scores differ"
        assert ok_cover
        assert nr > 0
