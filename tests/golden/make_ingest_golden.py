#!/usr/bin/env python3
"""Golden vectors for the device text loader, produced by the reference's own ``load_csv``.

Run in the build container (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_ingest_golden.py

Each case is a small text file (written verbatim to a temp dir), the loader arguments, and
what the UNMODIFIED reference (``countstream.database.load_csv``, database.py:171-207, and
``Database``, :36-84) returns for it: the (n, m) states and arities, or the exception type and
message.  The cases cover the grammar the reference's tests exercise (delimiter sniffing,
whitespace runs, blank lines, 1-based shift, ragged rows, non-integer tokens, negative states,
declared arities) plus the edges of str.splitlines / str.strip / int() the device tokeniser
has to reproduce (\\r\\n, lone \\r, \\v \\f \\x1c separators, signs, underscores, leading zeros,
empty fields, wide records).  Output: tests/golden/ingest_cases.json.
"""

from __future__ import annotations

import json
import os
import sys
import tempfile
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
sys.path.insert(0, "/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent

import numpy as np  # noqa: E402

from countstream.database import load_csv  # noqa: E402  (the reference)


def table(rows, sep=",", eol="\n"):
    return eol.join(sep.join(str(v) for v in r) for r in rows) + eol


def random_rows(seed, n, m, lo, hi):
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi, size=(m, n)).tolist()


def cases():
    c = []
    add = lambda name, text, delimiter=None, arities=None: c.append(  # noqa: E731
        {"name": name, "text": text, "delimiter": delimiter, "arities": arities})
    add("comma_0based", table(random_rows(1, 5, 40, 0, 4)))
    add("comma_1based", table(random_rows(2, 4, 30, 1, 4)))
    add("whitespace_runs", "  0 1\t2 \n\n1   0 2\t\n \t \n2 2 0\n")
    add("tabs_only", table(random_rows(3, 6, 25, 0, 3), sep="\t"))
    add("crlf", table(random_rows(4, 3, 20, 0, 5), eol="\r\n"))
    add("lone_cr", table(random_rows(5, 3, 20, 0, 5), eol="\r"))
    add("mixed_breaks", "0,1\x0b1,0\x0c1,1\x1c0,0\x1d1,1\x1e0,1\r\n1,0\r0,0\n")
    add("no_final_newline", "0 1 2\n2 1 0")
    add("spaces_around_fields", " 0 , 1 ,2\n1,  0,\t2 \n")
    add("signs_underscores_zeros", "+1,0_1,007\n-0,1_0,00\n")
    add("explicit_semicolon", table(random_rows(6, 4, 15, 0, 3), sep=";"), delimiter=";")
    add("explicit_tab", table(random_rows(7, 4, 15, 0, 3), sep="\t"), delimiter="\t")
    add("explicit_space_single", "0 1 1\n1 0 1\n", delimiter=" ")
    add("whitespace_vt_ff_sep", "0\x0c1\x1f2\n1 0\x1f2\n")
    add("declared_arities", table(random_rows(8, 3, 20, 0, 2)), arities=[2, 5, 3])
    add("single_column", "3\n1\n2\n0\n")
    add("single_value", "1\n")
    add("arity_256", table([[0, 255], [255, 0], [7, 9]]))
    add("arity_256_1based", table([[1, 256], [256, 1], [7, 9]]))
    add("wide_record", table(random_rows(9, 3000, 40, 0, 3)))
    add("very_wide_record", table(random_rows(10, 7000, 8, 0, 2)))
    add("many_rows", table(random_rows(11, 7, 5000, 0, 6)))
    add("leading_blank_lines", "\n\n  \n0,1\n1,0\n\n")
    # errors (DatabaseLoadError unless noted)
    add("err_empty", "")
    add("err_blank_only", "\n  \n\t\n")
    add("err_ragged", "0,1,2\n1,0\n2,2,2\n")
    add("err_ragged_longer", "0 1\n1 0 2\n")
    add("err_non_integer", "0,1\n1,x\n")
    add("err_empty_field", "0,,1\n1,0,1\n")
    add("err_trailing_comma", "0,1,\n1,0,1\n")
    add("err_double_underscore", "1__2,0\n0,1\n")
    add("err_leading_underscore", "_1,0\n0,1\n")
    add("err_float", "0,1.0\n1,0\n")
    add("err_sign_only", "0,-\n1,0\n")
    add("err_ragged_before_token", "0,1\n1,y,2\n")
    add("err_token_then_ragged", "0,1\nq,1\n1\n")
    add("err_negative", "0,1\n-1,0\n")
    add("err_declared_short", "0,1\n1,3\n", arities=[2, 2])
    add("err_declared_count", "0,1\n1,0\n", arities=[2, 2, 2])
    add("err_declared_zero", "0,0\n0,0\n", arities=[1, 0])
    return c


def main() -> None:
    out = []
    with tempfile.TemporaryDirectory() as td:
        for i, case in enumerate(cases()):
            p = Path(td) / f"c{i}.csv"
            p.write_bytes(case["text"].encode("latin-1"))
            rec = dict(case)
            try:
                db = load_csv(p, delimiter=case["delimiter"], arities=case["arities"])
                rec["data"] = np.asarray(db.data).tolist()
                rec["expect_arities"] = np.asarray(db.arities).tolist()
            except Exception as e:  # the reference's exception, recorded verbatim
                rec["error"] = type(e).__name__
                rec["message"] = str(e).replace(str(p), "{path}")
            out.append(rec)
    (HERE / "ingest_cases.json").write_text(json.dumps(out))
    print(f"wrote {len(out)} cases, {sum('error' in r for r in out)} errors")


if __name__ == "__main__":
    main()
