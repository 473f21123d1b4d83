"""TEST INFRASTRUCTURE ONLY -- numpy twin of the device column generator (k_generate).

Recomputes any rows of a device-generated column so the oracle can check
device counts on the same data without the device:

    key      = mix64(seed ^ mix64(0x632BE59BD9B4E019 + var))          (splitmix64 finaliser)
    u(row)   = mix64(key + row) >> 32                                   (row = global row id)
    pcfg     = sum_t state(parents[t], row) * prod_{u<t} arity(parents[u])
    state    = #{ t < r-1 : u >= thresholds[pcfg*(r-1) + t] }

(paper_1804_04640_b200/csrc/cs_common.cuh: mix64 / column_key / hash32;
 cs_kernels.cuh: k_generate.)
"""

from __future__ import annotations

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)
_K = np.uint64(0x632BE59BD9B4E019)


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _G
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def column_key(seed: int, var: int) -> np.uint64:
    with np.errstate(over="ignore"):
        inner = mix64(np.array([_K + np.uint64(var)], dtype=np.uint64))[0]
        return mix64(np.array([np.uint64(seed & (2**64 - 1)) ^ inner], dtype=np.uint64))[0]


def hash32(key: np.uint64, rows: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        return (mix64(np.uint64(key) + rows.astype(np.uint64)) >> np.uint64(32)).astype(np.uint32)


def generate_column(seed: int, var: int, r: int, thresholds, rows: np.ndarray,
                    parent_cols=(), parent_arities=()) -> np.ndarray:
    """States of `var` at global `rows`; parent_cols are the parents' states at those rows."""
    u = hash32(column_key(seed, var), np.asarray(rows, dtype=np.int64))
    thr = np.asarray(thresholds, dtype=np.uint32)
    rm1 = r - 1
    if rm1 == 0:
        return np.zeros(len(u), dtype=np.uint8)
    pcfg = np.zeros(len(u), dtype=np.int64)
    s = 1
    for pc, pr in zip(parent_cols, parent_arities):
        pcfg += pc.astype(np.int64) * s
        s *= int(pr)
    th = thr.reshape(-1, rm1)[pcfg]  # (rows, r-1)
    return (u[:, None] >= th).sum(axis=1).astype(np.uint8)


def generate_workload_columns(w, rows: np.ndarray, variables=None) -> dict:
    """Columns of a Workload (paper_1804_04640_b200.workloads) at `rows` -> {var: uint8[]}.

    Generator parents are materialised on demand (they always precede their child).
    """
    want = sorted(set(range(w.n) if variables is None else variables))
    out: dict = {}

    def col(v):
        if v not in out:
            ps = w.gen_parents[v]
            pcs = [col(p) for p in ps]
            out[v] = generate_column(w.seed, v, int(w.arities[v]), w.gen_thresholds[v], rows, pcs,
                                     [int(w.arities[p]) for p in ps])
        return out[v]

    for v in want:
        col(v)
    return {v: out[v] for v in want}
