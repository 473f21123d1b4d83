"""CLI: the reference's interface (argparse surface, JSONL schema, exit codes).

CPU: usage errors exit 2, data errors exit 1 with a JSON error on stderr, and without a GPU
the `gpu` strategy build is reported as a build_failure (exit 1) -- never silently computed on
the CPU.  GPU: the reference's binding golden cases replayed through the CLI.
"""

from __future__ import annotations

import json

import pytest

from paper_1804_04640_b200 import cli


def _lines(path):
    return [json.loads(x) for x in path.read_text().splitlines() if x.strip()]


def test_usage_errors_exit_2():
    with pytest.raises(SystemExit) as e:
        cli.main(["query"])
    assert e.value.code == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["query", "--target", "0", "--strategy", "radix"])
    assert e.value.code == 2


def test_data_errors_exit_1(tmp_path, capsys):
    assert cli.main(["query", "--target", "0"]) == 1
    err = json.loads(capsys.readouterr().err.strip())
    assert err["type"] == "error" and "--input or --synthetic" in err["message"]
    assert cli.main(["query", "--synthetic", "n=3,m=10,arity=2", "--target", "7"]) == 1
    assert "out of range" in json.loads(capsys.readouterr().err.strip())["message"]


def test_no_gpu_is_a_build_failure(tmp_path):
    import paper_1804_04640_b200._native as N

    if N.device_count() > 0:
        pytest.skip("a GPU is visible")
    out = tmp_path / "o.jsonl"
    rc = cli.main(["query", "--synthetic", "n=3,m=10,arity=2", "--target", "0", "--out", str(out)])
    assert rc == 1
    (line,) = _lines(out)
    assert line["type"] == "build_failure" and line["strategy"] == "gpu"


@pytest.mark.gpu
def test_golden_cases_through_cli(tmp_path, reference_cases):
    from conftest import rel_close

    for name, case in reference_cases.items():
        src = case["source"]
        if "csv" in src:
            f = tmp_path / "fixture.csv"
            f.write_text("\n".join(",".join(str(v + 1) for v in row) for row in zip(*case["data"])) + "\n")
            dbargs = ["--input", str(f)]
        else:
            a = src["arity"]
            part = f"{a[0]}-{a[1]}" if isinstance(a, list) else str(a)
            dbargs = ["--synthetic", f"n={src['n']},m={src['m']},arity={part},seed={src['seed']}"]
        for q in case["queries"]:
            base = dbargs + ["--target", str(q["target"])]
            if q["parents"]:
                base += ["--parents", ",".join(map(str, q["parents"]))]
            out = tmp_path / "r.jsonl"
            assert cli.main(["query", *base, "--agg", "records", "--out", str(out)]) == 0
            recs = [{k: r[k] for k in ("config", "k", "n_ijk", "n_ij")} for r in _lines(out) if r["type"] == "record"]
            assert sorted(recs, key=lambda r: (r["config"], r["k"])) == q["records"], name
            for agg in ("loglik", "mdl"):
                assert cli.main(["query", *base, "--agg", agg, "--out", str(out)]) == 0
                (score,) = [r for r in _lines(out) if r["type"] == "score"]
                assert rel_close(score["value"], q[agg], 1e-9), (name, agg)
        out = tmp_path / "l.jsonl"
        assert cli.main(["learn-parents", *dbargs, "--max-parents", str(case["learn"]["maxParents"]),
                         "--out", str(out)]) == 0
        got = [r for r in _lines(out) if r["type"] == "parent_set"]
        assert [g["parents"] for g in got] == [p["parents"] for p in case["learn"]["parentSets"]], name
        if "rules" in case:
            rr = case["rules"]
            assert cli.main(["mine-rules", *dbargs, "--min-support", str(rr["minSupport"]), "--min-confidence",
                             str(rr["minConfidence"]), "--max-size", str(rr["maxSize"]), "--out", str(out)]) == 0
            got = sorted(([r["antecedent"], r["consequent"]] for r in _lines(out) if r["type"] == "rule"))
            assert got == sorted([r["antecedent"], r["consequent"]] for r in rr["rules"]), name


@pytest.mark.gpu
def test_device_ingest_cli_matches_host_loader(tmp_path, reference_cases):
    """`--device-ingest` (CSV tokenised on the GPU) gives the same JSONL as the host loader for
    every golden case's database written out as a 1-based CSV: records, scores, learned parent
    sets and rules."""
    import numpy as np

    from conftest import case_db

    for name, case in reference_cases.items():
        db = case_db(case)
        f = tmp_path / f"{name}.csv"
        f.write_text("\n".join(",".join(str(int(v) + 1) for v in row) for row in np.asarray(db.data).T) + "\n")
        outs = []
        for extra in ([], ["--device-ingest"]):
            dbargs = ["--input", str(f), *extra]
            res = []
            for q in case["queries"]:
                base = dbargs + ["--target", str(q["target"])]
                if q["parents"]:
                    base += ["--parents", ",".join(map(str, q["parents"]))]
                for agg in ("records", "loglik", "mdl"):
                    out = tmp_path / "q.jsonl"
                    assert cli.main(["query", *base, "--agg", agg, "--out", str(out)]) == 0
                    res.append([r for r in _lines(out) if r["type"] in ("record", "score")])
            out = tmp_path / "l.jsonl"
            assert cli.main(["learn-parents", *dbargs, "--max-parents", "2", "--out", str(out)]) == 0
            res.append([r["parents"] for r in _lines(out) if r["type"] == "parent_set"])
            outs.append(res)
        assert outs[0] == outs[1], name
