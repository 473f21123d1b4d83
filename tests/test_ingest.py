"""Device text ingest (cs_db_load_text) vs the reference's load_csv.

Golden cases: tests/golden/ingest_cases.json, recorded from the unmodified reference
(tests/golden/make_ingest_golden.py).  The CPU test pins this package's host restatement of
load_csv to them; the GPU tests require the device loader to reproduce every case byte for
byte (columns, arities) or raise the same exception with the same message, and check large
seeded files (many 16 KB text chunks, 1-based shift, device-resident input) against the
matrix they were printed from.
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN

CASES = json.loads((GOLDEN / "ingest_cases.json").read_text())


def _write(tmp_path, case):
    p = tmp_path / f"{case['name']}.csv"
    p.write_bytes(case["text"].encode("latin-1"))
    return p


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_host_load_csv_matches_reference(tmp_path, case):
    import paper_1804_04640_b200 as cs

    p = _write(tmp_path, case)
    if "error" in case:
        with pytest.raises(cs.DatabaseLoadError) as ei:
            cs.load_csv(p, delimiter=case["delimiter"], arities=case["arities"])
        assert str(ei.value) == case["message"].replace("{path}", str(p))
        return
    db = cs.load_csv(p, delimiter=case["delimiter"], arities=case["arities"])
    assert db.data.tolist() == case["data"]
    assert db.arities.tolist() == case["expect_arities"]


def _device_columns(ddb):
    return np.stack([ddb.gdb.download(i) for i in range(ddb.n)])


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_device_loader_matches_reference(tmp_path, case):
    import paper_1804_04640_b200 as cs

    p = _write(tmp_path, case)
    if "error" in case:
        with pytest.raises(cs.DatabaseLoadError) as ei:
            cs.load_csv_device(p, delimiter=case["delimiter"], arities=case["arities"])
        assert str(ei.value) == case["message"].replace("{path}", str(p))
        return
    ddb = cs.load_csv_device(p, delimiter=case["delimiter"], arities=case["arities"])
    want = np.asarray(case["data"], dtype=np.int64)
    assert (ddb.n, ddb.m) == want.shape
    assert np.array_equal(_device_columns(ddb), want.astype(np.uint8))
    assert ddb.arities.tolist() == case["expect_arities"]


def _big_text(rng, m, arities, sep, one_based, blank_every=0):
    x = np.stack([rng.integers(0, a, size=m) for a in arities]).astype(np.int64)
    rows = (x.T + (1 if one_based else 0)).astype(str)
    lines = [sep.join(r) for r in rows]
    if blank_every:
        lines = [ln if i % blank_every else ln + "\n  " for i, ln in enumerate(lines)]
    return x, ("\n".join(lines) + "\n").encode()


@pytest.mark.gpu
@pytest.mark.parametrize("sep,one_based", [(",", False), (" ", True), ("\t", False)])
def test_device_loader_large(sep, one_based):
    import paper_1804_04640_b200 as cs
    from paper_1804_04640_b200.engine import GpuDatabase

    rng = np.random.default_rng(7)
    arities = [2, 3, 4, 5, 8, 16, 17, 100, 2, 3, 4, 5, 6, 7, 250, 2]
    x, text = _big_text(rng, 400_000, arities, sep, one_based, blank_every=9973)
    gdb = GpuDatabase.from_text(cs.shared_context(0), text)
    assert (gdb.n, gdb.m) == x.shape
    got = np.stack([gdb.download(i) for i in range(gdb.n)])
    assert np.array_equal(got, x.astype(np.uint8))
    assert gdb.arities.tolist() == (x.max(axis=1) + 1).tolist()
    assert gdb.load_info["one_based"] == one_based


@pytest.mark.gpu
def test_device_loader_device_input_and_queries():
    """Text already in HBM (torch CUDA tensor) -> database -> counting queries through the
    drop-in strategy agree with the host Database built from the same matrix."""
    import torch

    import paper_1804_04640_b200 as cs
    from paper_1804_04640_b200.engine import GpuDatabase

    rng = np.random.default_rng(11)
    arities = [3, 2, 4, 3, 5, 2]
    x, text = _big_text(rng, 200_000, arities, ",", False)
    dev = torch.frombuffer(bytearray(text), dtype=torch.uint8).cuda()
    gdb = GpuDatabase.from_text(cs.shared_context(0), dev)
    ddb = cs.DeviceDatabase(gdb)
    host = cs.Database(x, arities)
    s_dev = cs.GpuStrategy(ddb)
    s_host = cs.GpuStrategy(host)
    for q in [cs.QuerySpec(0, (1, 2)), cs.QuerySpec(4, (5, 3, 1)), cs.QuerySpec(2, ())]:
        a, b = cs.LogLikelihood(), cs.LogLikelihood()
        s_dev.query(q, a)
        s_host.query(q, b)
        assert a.result() == b.result()
        r1, r2 = cs.RecordCollector(), cs.RecordCollector()
        s_dev.query(q, r1)
        s_host.query(q, r2)
        assert r1.result() == r2.result()


@pytest.mark.gpu
def test_device_loader_unsupported():
    import paper_1804_04640_b200 as cs
    from paper_1804_04640_b200.engine import GpuDatabase

    with pytest.raises(cs.UnsupportedQueryError):
        GpuDatabase.from_text(cs.shared_context(0), b"0,300\n1,2\n")
    with pytest.raises(cs.UnsupportedQueryError):
        GpuDatabase.from_text(cs.shared_context(0), b"0;;1\n", delimiter=";;")
