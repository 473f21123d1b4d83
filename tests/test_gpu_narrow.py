"""The narrow-counter SMEM class (8 / 16-bit counters with exact wrap repair, cs_kernels.cuh
hist_smem_narrow): tables of 56K..225K cells counted in SMEM instead of by the partition class.
Parity against the dense oracle on uniform data, and on skewed data whose counters wrap
hundreds of times per cell (carries across the lanes of a word)."""

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


@pytest.mark.parametrize("m", [1000, 65_537, 2_000_003])
def test_narrow_uniform(ctx, monkeypatch, capfd, m):
    rng = np.random.default_rng(m)
    ar = [16, 15, 13, 16, 8, 7, 9, 5]
    data = np.vstack([rng.integers(0, a, m) for a in ar]).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, ar)
    # 16*15*13 = 3120 .. 16*15*13*16 = 49,920 (SMEM) | *8 = 399K (spill / partition) ...
    qs = [(0, 1, 2, 5, 7), (0, 1, 2, 4, 7), (3, 2, 1, 0), (1, 3, 4, 5), (0, 3, 5, 6), (2, 3, 6, 7, 4),
          (0, 1, 3, 4), (5, 0, 1, 2, 6), (7, 6, 5, 4, 3, 2)]
    monkeypatch.setenv("CS_TRACE", "1")
    _check(gdb, data, ar, qs)
    cls = _classes(capfd)
    assert cls["smem"] >= 4 and cls["partition"] + cls["spill"] >= 1
    monkeypatch.setenv("CS_NARROW_SEG_ROWS", "65536")  # many segments per query
    monkeypatch.setenv("CS_SEG_MAX_ROWS", "65536")
    _check(gdb, data, ar, qs)
    monkeypatch.setenv("CS_NARROW_FAST", "0")  # no optimistic pass: the exact form alone
    _check(gdb, data, ar, qs)


@pytest.mark.parametrize("fast", ["1", "0"])
@pytest.mark.parametrize("skew", ["constant", "four_lanes", "two_cells_far"])
def test_narrow_wraps(ctx, monkeypatch, skew, fast):
    """Counters wrap many times: one constant cell (carry out of lane 3 / the high half), rows
    cycling through the 4 lanes of one word (carries through every lane), two hot cells.  With
    the optimistic pass on (fast = 1) its counter-sum check must catch every one of these and
    fall back to the exact form."""
    monkeypatch.setenv("CS_NARROW_FAST", fast)
    m = 3_000_017
    ar = [16, 16, 16, 13]  # 53,248 cells: 32-bit class; with a 5th digit -> narrow
    ar5 = ar + [3]
    rng = np.random.default_rng(1)
    data = np.zeros((5, m), dtype=np.uint8)
    if skew == "four_lanes":
        data[0] = np.arange(m) % 4  # cells 0..3 = lanes 0..3 of word 0 (8-bit) / words 0-1 (16-bit)
    elif skew == "two_cells_far":
        hot = rng.random(m) < 0.5
        data[:, hot] = np.array([15, 15, 15, 12, 2], dtype=np.uint8)[:, None]  # the last cell
    data[4, rng.random(m) < 0.001] = 1  # a sprinkle elsewhere
    gdb = GpuDatabase.from_columns(ctx, data, ar5)
    qs = [(0, 1, 2, 3, 4), (4, 3, 2, 1, 0), (1, 0, 2, 3, 4)]  # 159,744 cells: 8-bit counters
    qs16 = [(0, 1, 2, 3), (0, 1, 3, 4, 2)]  # 53,248 (32-bit) and 79,872 cells (16-bit)
    _check(gdb, data, ar5, qs + qs16)
    monkeypatch.setenv("CS_NARROW_SEG_ROWS", "262144")
    monkeypatch.setenv("CS_SEG_MAX_ROWS", "262144")
    _check(gdb, data, ar5, qs + qs16)


def test_narrow_off_matches_partition(ctx, monkeypatch):
    rng = np.random.default_rng(9)
    m = 1_000_000
    ar = [8] * 6
    data = rng.integers(0, 8, (6, m)).astype(np.uint8)
    gdb = GpuDatabase.from_columns(ctx, data, ar)
    qs = [tuple(int(x) for x in rng.permutation(6)) for _ in range(20)]  # 262,144 cells: partition
    qs += [tuple(int(x) for x in rng.permutation(6)[:5]) + () for _ in range(4)]  # 32,768: SMEM
    qs += [(0, 1, 2, 3, 4, 5)[:6]]
    monkeypatch.setenv("CS_NARROW", "0")
    monkeypatch.setenv("CS_SPILL", "0")
    _check(gdb, data, ar, qs)
    monkeypatch.setenv("CS_NARROW", "1")
    ar2 = [8, 8, 8, 8, 8, 3]
    data2 = data.copy()
    data2[5] %= 3
    gdb2 = GpuDatabase.from_columns(ctx, data2, ar2)
    qs2 = [(0, 1, 2, 3, 4, 5), (5, 4, 3, 2, 1, 0)]  # 98,304 cells: 16-bit narrow
    _check(gdb2, data2, ar2, qs2)


@pytest.mark.parametrize("m", [70_001, 4_500_000])
def test_narrow_multipass(ctx, monkeypatch, capfd, m):
    """Tables above 4x the SMEM capacity in several cell-range passes (CS_NARROW_MAX_PASSES):
    uniform cells plus a hot cell whose 8-bit counter wraps in every pass's range."""
    monkeypatch.setenv("CS_NARROW_MAX_PASSES", "8")
    monkeypatch.setenv("CS_TRACE", "1")
    rng = np.random.default_rng(m)
    ar = [16, 16, 16, 16, 6, 5]
    data = np.vstack([rng.integers(0, a, m) for a in ar]).astype(np.uint8)
    hot = rng.random(m) < 0.3
    data[:, hot] = np.array([3, 1, 4, 1, 5, 2], dtype=np.uint8)[:, None]
    gdb = GpuDatabase.from_columns(ctx, data, ar)
    qs = [(0, 1, 2, 3, 4), (4, 3, 2, 1, 0), (0, 1, 2, 3, 5), (5, 0, 1, 2, 3), (1, 2, 3, 4, 5)]
    _check(gdb, data, ar, qs)  # 393,216 / 327,680 / 122,880 cells: 2 passes, 2 passes, 1
    c = _classes(capfd)
    assert c["partition"] == 0 and c["spill"] == 0
    monkeypatch.setenv("CS_NARROW_PASS_SEG_ROWS", "65536")
    _check(gdb, data, ar, qs)
