"""The spill class (cs_spill.cuh): tables of 225K .. ~600K cells.  k_spill_hist counts the first
220K cells in SMEM and appends every other row's index to a warp-private stream; k_spill_count
finishes the 192K-cell groups past them.  Parity against the dense oracle on uniform data, ragged and
tiny m, forced segmentation and one-query waves, regions too small for their rows (the overflow
rows go to the global table one by one), and hot cells whose 8-bit counters wrap in both kernels."""

from __future__ import annotations

import numpy as np
import pytest

import oracle as O
from conftest import rel_close

pytestmark = pytest.mark.gpu

import paper_1804_04640_b200 as cs  # noqa: E402
from paper_1804_04640_b200._native import CS_WANT_TABLES  # noqa: E402
from paper_1804_04640_b200.engine import GpuDatabase, QueryPlan  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    return cs.shared_context(0)


def _classes(capfd):
    err = capfd.readouterr().err
    line = [x for x in err.splitlines() if "plan_build: classes" in x][-1]
    return {kv.split("=")[0]: int(kv.split("=")[1]) for kv in line.split("classes ")[1].split()}


def _check(gdb, data, ar, qs, mi=True):
    plan = QueryPlan(gdb, qs, CS_WANT_TABLES)
    tabs = np.zeros(plan.total_cells, dtype=np.uint32)
    ll, miv = np.zeros(plan.nq), np.zeros(plan.nq)
    nnz = np.zeros(plan.nq, dtype=np.int64)
    plan.execute(tables=tabs, loglik=ll, mi=miv if mi else None, nnz=nnz)
    plan.close()
    otabs, _, oll, omi, onnz = O.dense_tables(data, ar, qs)
    bad = np.flatnonzero(tabs != otabs)
    assert bad.size == 0, f"{bad.size} cells differ, first {bad[:5]}: {tabs[bad[:5]]} vs {otabs[bad[:5]]}"
    assert np.array_equal(nnz, onnz)
    assert all(rel_close(a, b, 1e-9) for a, b in zip(ll, oll))
    if mi:
        m = data.shape[1]
        assert np.all(np.abs(miv - omi) <= 1e-9 * (np.abs(oll) + 1) / m + 1e-15)


AR = [16, 15, 13, 16, 8, 7, 9, 5]
# cells (192K-cell groups past the first 220K): 399,360 (1) x 2, 349,440 (1) x 2, 449,280 (2), 249,600 (1),
# 604,800 (2) x 2, 524,160 (2) x 2, 604,800 (2), 524,160 (2), 873,600 (4: partition class unless
# CS_SPILL_GROUPS >= 4); then 7,862,400 (partition class) and 67,200 (narrow class)
QS = [(0, 1, 2, 3, 4), (4, 3, 2, 1, 0), (0, 1, 2, 3, 5), (5, 3, 1, 0, 2), (0, 1, 2, 3, 6), (7, 0, 1, 2, 3),
      (1, 3, 4, 5, 6, 7), (0, 4, 5, 6, 7, 1), (2, 4, 5, 6, 7, 0), (4, 5, 6, 7, 2, 3), (4, 5, 7, 0, 1, 6),
      (7, 6, 5, 4, 3, 2), (0, 1, 2, 4, 5, 7), (4, 7, 5, 6, 2, 1, 0), (7, 4, 5, 0, 1)]


@pytest.mark.parametrize("m", [1, 33, 1000, 65_537, 2_000_003])
def test_spill_uniform(ctx, monkeypatch, capfd, m):
    rng = np.random.default_rng(m + 1)
    data = np.vstack([rng.integers(0, a, m) for a in AR]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, AR)
    monkeypatch.setenv("CS_TRACE", "1")
    _check(gdb, data, AR, QS)
    cls = _classes(capfd)
    assert cls["spill"] == 12 and cls["partition"] == 2 and cls["smem"] == 1
    monkeypatch.setenv("CS_SPILL_SEG_ROWS", "65536")  # many segments per query
    monkeypatch.setenv("CS_SPILL_MB", "1")            # one query per wave
    _check(gdb, data, AR, QS)
    monkeypatch.setenv("CS_SPILL_GROUPS", "1")        # tables above 220K + 192K cells: partition class
    _check(gdb, data, AR, QS)
    cls = _classes(capfd)
    assert cls["spill"] == 5 and cls["partition"] == 9
    monkeypatch.setenv("CS_SPILL_GROUPS", "4")        # up to 220K + 768K cells
    _check(gdb, data, AR, QS)
    cls = _classes(capfd)
    assert cls["spill"] == 13 and cls["partition"] == 1
    monkeypatch.setenv("CS_STREAMS", "1")             # every launch on the context stream
    _check(gdb, data, AR, QS)
    monkeypatch.setenv("CS_NARROW_FAST", "0")         # optimistic passes always followed by the exact recount
    _check(gdb, data, AR, QS)


@pytest.mark.parametrize("slack", ["0", "50", "125"])
@pytest.mark.parametrize("skew", ["hot_spill", "hot_direct", "lanes"])
def test_spill_skewed_and_overflow(ctx, monkeypatch, slack, skew):
    """Streams switched off (slack 0: every spilled row goes to the table), sized at half of and
    above the uniform expectation;
    30% of the rows in one cell of a spill range (its counter wraps ~4,000 times in
    k_spill_count, or overflows to the table), in one cell of the SMEM range, or cycling through
    the four lanes of one counter word of a spill range."""
    m = 3_500_017
    rng = np.random.default_rng(11)
    data = np.vstack([rng.integers(0, a, m) for a in AR]).astype(np.uint8)
    hot = rng.random(m) < 0.3
    if skew == "hot_spill":
        data[:, hot] = np.array([15, 14, 12, 15, 7, 6, 8, 4], dtype=np.uint8)[:, None]  # the last cell
    elif skew == "hot_direct":
        data[:, hot] = np.array([3, 1, 4, 1, 0, 0, 0, 0], dtype=np.uint8)[:, None]
    else:
        data[:, hot] = np.array([0, 0, 0, 0, 7, 6, 8, 4], dtype=np.uint8)[:, None]
        data[0, hot] = (np.arange(int(hot.sum())) % 4).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, AR)
    monkeypatch.setenv("CS_SPILL_SLACK", slack)
    monkeypatch.setenv("CS_SPILL_GROUPS", "4")
    qs = QS[:4] + QS[6:8] + QS[12:13]
    _check(gdb, data, AR, qs)
    monkeypatch.setenv("CS_SPILL_SEG_ROWS", "524288")
    _check(gdb, data, AR, qs, mi=False)
    if slack == "125":
        # the same skewed tables through the partition class
        monkeypatch.setenv("CS_SPILL", "0")
        _check(gdb, data, AR, qs, mi=False)


def test_spill_matches_partition_class(ctx, monkeypatch):
    """The same batch through the spill class and through the partition class it replaces."""
    rng = np.random.default_rng(5)
    m = 1_200_000
    data = np.vstack([rng.integers(0, a, m) for a in AR]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, AR)
    out = []
    for spill in ("1", "0"):
        monkeypatch.setenv("CS_SPILL", spill)
        plan = QueryPlan(gdb, QS, CS_WANT_TABLES)
        tabs = np.zeros(plan.total_cells, dtype=np.uint32)
        ll = np.zeros(plan.nq)
        plan.execute(tables=tabs, loglik=ll)
        plan.close()
        out.append((tabs, ll))
    assert np.array_equal(out[0][0], out[1][0])
    assert all(rel_close(a, b, 1e-12) for a, b in zip(out[0][1], out[1][1]))
