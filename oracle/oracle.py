"""TEST INFRASTRUCTURE ONLY -- the parity oracle.  Never imported by the product package.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may use this module, and only as the checker or as the
timed CPU baseline.

Two restatements of the reference counting path (reference = countstream,
/root/reference/pkg/src/countstream):

* numpy, definitional -- :func:`oracle_records` restates ``oracle_query``
  (oracle.py:19-56: one boolean mask per candidate parent configuration,
  candidates narrowed to observed configurations past ``exhaustive_limit``)
  and :func:`oracle_count` restates ``oracle_count`` (oracle.py:59-65);
* C, algorithmic -- :func:`radix_tables` drives ``radix_oracle.c``, the
  level-wise radix partition of ``radix_query`` (radix.py:33-156), multi-threaded
  over queries; it is the CPU baseline and the oracle at sizes where masks are slow.
* C, direct -- :func:`dense_tables` (``count_oracle.c``): the joint-key convention of
  ``_config_keys`` (baselines.py:51-57) counted into a dense table, then LL / MI / nnz;
  :func:`itemset_supports_enum`: all 2-/3-itemset supports counted record by record.  Used
  by the full-size parity tests, where the radix port would take minutes.

Pinned by tests/test_oracle_golden.py against golden vectors generated from the
reference itself (tests/golden/make_golden.py) and the reference's hand-derived KATs.
"""

from __future__ import annotations

import ctypes
import itertools
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "libradix_oracle.so"


def build() -> Path:
    """Compile radix_oracle.c (gcc) into oracle/_build/."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        lib.oracle_radix_tables.restype = ctypes.c_int
        lib.oracle_radix_tables.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_int32, P, P, P,
                                            P, P, P, ctypes.c_int32]
        lib.oracle_bitmap_pack.restype = None
        lib.oracle_bitmap_pack.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P]
        lib.oracle_dense_tables.restype = ctypes.c_int
        lib.oracle_dense_tables.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_int32, P, P, P,
                                            P, P, P, P, ctypes.c_int32]
        lib.oracle_itemset_enum.restype = ctypes.c_int
        lib.oracle_itemset_enum.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int32, P, P,
                                            ctypes.c_int32]
        lib.oracle_bitmap_counts.restype = ctypes.c_int
        lib.oracle_bitmap_counts.argtypes = [P, P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, P,
                                             ctypes.c_int32]
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


# ---------------------------------------------------------------------------------------------
# definitional numpy oracle


def oracle_records(data: np.ndarray, arities, target: int, parents, exhaustive_limit: int = 4096) -> set:
    """Non-zero cells of query (target | parents) as a set of (config, k, n_ijk, n_ij) tuples.

    Restates reference oracle.py:19-56.  ``data`` is (n, m) with row i = variable i.
    ``config`` is ((var, state), ...) sorted by variable.
    """
    parents = tuple(int(p) for p in parents)
    tcol = data[target]
    r_t = int(arities[target])
    space = 1
    for p in parents:
        space *= int(arities[p])
    if space <= exhaustive_limit:
        cands = itertools.product(*(range(int(arities[p])) for p in parents))
    else:
        obs = np.unique(np.ascontiguousarray(data[list(parents)].T), axis=0)
        cands = (tuple(int(s) for s in row) for row in obs)
    out = set()
    m = data.shape[1]
    for states in cands:
        mask = np.ones(m, dtype=bool)
        for p, s in zip(parents, states):
            mask &= data[p] == s
        n_ij = int(mask.sum())
        if n_ij == 0:
            continue
        config = tuple(sorted(zip(parents, states)))
        hits = tcol[mask]
        for k in range(r_t):
            c = int(np.count_nonzero(hits == k))
            if c:
                out.add((config, k, c, n_ij))
    return out


def oracle_count(data: np.ndarray, variables, states) -> int:
    """Records matching every (var, state) pair (reference oracle.py:59-65)."""
    mask = np.ones(data.shape[1], dtype=bool)
    for v, s in zip(variables, states):
        mask &= data[v] == s
    return int(mask.sum())


def loglik_of_records(records) -> float:
    """Direct sum N_ijk ln(N_ijk/N_ij) (reference tests conftest.py:97-99 loglik_direct)."""
    return math.fsum(r[2] * math.log(r[2] / r[3]) for r in records)


def mdl_of(ll: float, m: int, r_i: int, q_i: int) -> float:
    """MdlScore.result (aggregators.py:191-193)."""
    return -ll + 0.5 * math.log(m) * (r_i - 1) * q_i


def mi_of_records(records, m: int) -> float:
    """I(X;Pa) = (1/m) sum n ln(m n / (n_ij n_k)) in fp64 (survey 8a definition)."""
    if not records:
        return 0.0
    nk: dict = {}
    for _, k, n, _ in records:
        nk[k] = nk.get(k, 0) + n
    return math.fsum(n * math.log(m * n / (nij * nk[k])) for _, k, n, nij in records) / m


def table_from_records(records, target: int, parents, arities) -> np.ndarray:
    """Dense uint32 table in the engine's joint-index order (target least significant)."""
    r_t = int(arities[target])
    strides = {}
    s = r_t
    for p in parents:
        strides[p] = s
        s *= int(arities[p])
    t = np.zeros(s, dtype=np.uint32)
    for config, k, n, _ in records:
        idx = k + sum(st * strides[v] for v, st in config)
        t[idx] = n
    return t


def records_from_table(table: np.ndarray, target: int, parents, arities) -> set:
    """Inverse of :func:`table_from_records`."""
    r_t = int(arities[target])
    parents = tuple(parents)
    t = np.asarray(table).reshape(-1, r_t).astype(np.int64)
    nij = t.sum(axis=1)
    out = set()
    for j, k in zip(*np.nonzero(t)):
        rem = int(j)
        cfg = []
        for p in parents:
            rem, s = divmod(rem, int(arities[p]))
            cfg.append((p, s))
        out.add((tuple(sorted(cfg)), int(k), int(t[j, k]), int(nij[j])))
    return out


# ---------------------------------------------------------------------------------------------
# C radix restatement


def radix_tables(cols_u8: np.ndarray, arities, queries, nthreads: int | None = None,
                 want_tables: bool = True):
    """Run the radix restatement over ``queries`` (variable tuples, target first).

    Returns (tables uint32 packed | None, table_off int64, loglik float64, nnz int64).
    """
    lib = _load()
    cols = np.ascontiguousarray(cols_u8, dtype=np.uint8)
    n, m = cols.shape
    ar = np.ascontiguousarray(arities, dtype=np.int32)
    qs = [tuple(int(v) for v in q) for q in queries]
    off = np.zeros(len(qs) + 1, dtype=np.int32)
    off[1:] = np.cumsum([len(q) for q in qs]) if qs else []
    flat = np.array([v for q in qs for v in q], dtype=np.int32)
    cells = np.array([int(np.prod([int(ar[v]) for v in q], dtype=np.int64)) for q in qs], dtype=np.int64)
    toff = np.zeros(len(qs), dtype=np.int64)
    if len(qs):
        toff[1:] = np.cumsum(cells)[:-1]
    tables = np.zeros(int(cells.sum()), dtype=np.uint32) if want_tables else None
    ll = np.zeros(len(qs))
    nnz = np.zeros(len(qs), dtype=np.int64)
    nt = nthreads or os.cpu_count() or 1
    if qs:
        rc = lib.oracle_radix_tables(_p(cols), m, m, _p(ar), len(qs), _p(off), _p(flat), _p(toff),
                                     _p(tables), _p(ll), _p(nnz), nt)
        if rc != 0:
            raise RuntimeError(f"oracle_radix_tables failed: {rc}")
    return tables, toff, ll, nnz


def bitmap_planes(col_u8: np.ndarray, state: int) -> np.ndarray:
    """bitmap._pack restatement: uint32 words, bit t%32 of word t/32 = record t."""
    lib = _load()
    col = np.ascontiguousarray(col_u8, dtype=np.uint8)
    out = np.zeros((len(col) + 31) // 32, dtype=np.uint32)
    lib.oracle_bitmap_pack(_p(col), len(col), int(state), _p(out))
    return out


def bitmap_counts(planes: dict, itemsets, m: int, nthreads: int | None = None) -> np.ndarray:
    """bitmap_count restatement: popcount of the AND of planes[(var, state)] per itemset.

    ``itemsets`` is a list of ((var, state), ...) tuples.
    """
    lib = _load()
    keep = []
    ptrs = []
    off = [0]
    nwords = None
    for its in itemsets:
        for key in its:
            a = planes[key]
            nwords = len(a)
            keep.append(a)
            ptrs.append(a.ctypes.data)
        off.append(len(ptrs))
    arr = (ctypes.c_void_p * max(len(ptrs), 1))(*ptrs)
    offa = np.asarray(off, dtype=np.int32)
    out = np.zeros(len(itemsets), dtype=np.int64)
    lib.oracle_bitmap_counts(ctypes.cast(arr, ctypes.c_void_p), _p(offa), len(itemsets),
                             int(nwords or 0), int(m), _p(out), nthreads or os.cpu_count() or 1)
    return out


# ---------------------------------------------------------------------------------------------
# C direct-count restatements (count_oracle.c)


def _encode(queries):
    qs = [tuple(int(v) for v in q) for q in queries]
    off = np.zeros(len(qs) + 1, dtype=np.int32)
    if qs:
        off[1:] = np.cumsum([len(q) for q in qs])
    flat = np.array([v for q in qs for v in q], dtype=np.int32)
    return qs, off, flat


def dense_tables(cols_u8: np.ndarray, arities, queries, nthreads: int | None = None,
                 want_tables: bool = True, m: int | None = None):
    """Direct dense count of ``queries`` (variable tuples, target first) over the first ``m``
    rows of ``cols_u8`` (n x ld, default all).

    Returns (tables uint32 packed | None, table_off int64, loglik, mi, nnz).
    """
    lib = _load()
    cols = np.ascontiguousarray(cols_u8, dtype=np.uint8)
    n, ld = cols.shape
    m = ld if m is None else int(m)
    ar = np.ascontiguousarray(arities, dtype=np.int32)
    qs, off, flat = _encode(queries)
    cells = np.array([int(np.prod([int(ar[v]) for v in q], dtype=np.int64)) for q in qs], dtype=np.int64)
    toff = np.zeros(len(qs), dtype=np.int64)
    if len(qs):
        toff[1:] = np.cumsum(cells)[:-1]
    tables = np.zeros(int(cells.sum()), dtype=np.uint32) if want_tables else None
    ll = np.zeros(len(qs))
    mi = np.zeros(len(qs))
    nnz = np.zeros(len(qs), dtype=np.int64)
    if qs:
        rc = lib.oracle_dense_tables(_p(cols), ld, m, _p(ar), len(qs), _p(off), _p(flat), _p(toff),
                                     _p(tables), _p(ll), _p(mi), _p(nnz), nthreads or os.cpu_count() or 1)
        if rc != 0:
            raise RuntimeError(f"oracle_dense_tables failed: {rc}")
    return tables, toff, ll, mi, nnz


def itemset_supports_enum(item_cols: np.ndarray, nthreads: int | None = None, m: int | None = None):
    """(pairs (n, n) int64 with [a, b] for a < b, triples int64 in itertools.combinations order)
    of the n binary item columns (rows = items, state 1 = present)."""
    lib = _load()
    cols = np.ascontiguousarray(item_cols, dtype=np.uint8)
    n, ld = cols.shape
    m = ld if m is None else int(m)
    pairs = np.zeros((n, n), dtype=np.int64)
    triples = np.zeros(max(n * (n - 1) * (n - 2) // 6, 1), dtype=np.int64)
    rc = lib.oracle_itemset_enum(_p(cols), ld, m, n, _p(pairs), _p(triples), nthreads or os.cpu_count() or 1)
    if rc != 0:
        raise RuntimeError(f"oracle_itemset_enum failed: {rc}")
    return pairs, triples[: n * (n - 1) * (n - 2) // 6]
