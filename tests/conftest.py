"""Shared test helpers.

Markers: ``gpu`` = needs a B200 (run with ``-m gpu`` on the GPU box); everything
else runs on the CPU build container (``-m "not gpu"``).

The oracle (``oracle/``) is test infrastructure: tests import it as the checker.
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


@pytest.fixture(scope="session")
def reference_cases() -> dict:
    return json.loads((GOLDEN / "reference_cases.json").read_text())


@pytest.fixture(scope="session")
def random_sweep() -> dict:
    with gzip.open(GOLDEN / "random_sweep.json.gz", "rt") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def cfg1_golden() -> dict:
    z = np.load(GOLDEN / "cfg1.npz")
    return {k: z[k] for k in z.files}


def golden_records(q: dict) -> set:
    """Golden JSON records -> set of (config, k, n_ijk, n_ij) tuples."""
    return {(tuple(tuple(c) for c in r["config"]), r["k"], r["n_ijk"], r["n_ij"]) for r in q["records"]}


def case_db(case: dict):
    """Rebuild a golden case's database with this package's (restated) loaders."""
    from paper_1804_04640_b200.database import Database, generate_synthetic, parse_synthetic

    src = case["source"]
    if "data" in case:
        return Database(np.array(case["data"], dtype=np.int32), case["arities"])
    if "csv" in src:
        raise KeyError("csv case without inline data")
    a = src["arity"]
    part = f"{a[0]}-{a[1]}" if isinstance(a, list) else str(a)
    return parse_synthetic(f"n={src['n']},m={src['m']},arity={part},seed={src['seed']}")


def sweep_db(d: dict):
    from paper_1804_04640_b200.database import generate_synthetic

    return generate_synthetic(d["n"], d["m"], d["arities"], seed=d["seed"])


def rel_close(a: float, b: float, rel: float = 1e-9, abs_: float = 1e-12) -> bool:
    return abs(a - b) <= max(rel * max(abs(a), abs(b)), abs_)


# hand-derived KATs of the reference's own tests (pkg/tests/test_oracle.py:19-27, 37-40, 61-74)
FIXTURE_X1_GIVEN_X0_X2 = {
    (((0, 0), (2, 0)), 0, 1, 2),
    (((0, 0), (2, 0)), 1, 1, 2),
    (((0, 1), (2, 0)), 0, 1, 2),
    (((0, 1), (2, 0)), 1, 1, 2),
    (((0, 1), (2, 1)), 0, 1, 1),
    (((0, 2), (2, 0)), 1, 2, 2),
    (((0, 2), (2, 1)), 0, 1, 1),
}
FIXTURE_X2_EMPTY = {((), 0, 6, 8), ((), 1, 2, 8)}
# 1-based fixture rows as stored in the reference's tests/data/fixture.csv (conftest.py:33-36)
FIXTURE_ROWS_1BASED = [
    (1, 1, 1), (1, 2, 1), (2, 1, 2), (2, 2, 1),
    (3, 2, 1), (3, 2, 1), (3, 1, 2), (2, 1, 1),
]
