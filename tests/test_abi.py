"""The C ABI library loads on a CPU-only host and exports every symbol include/*.h declares.

No compute calls (there is no GPU here); the only calls are ones that must fail cleanly
without a device.
"""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

from conftest import ROOT

HEADER = ROOT / "include" / "countstream_gpu.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(cs_\w+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("cs_ctx_create", "cs_db_create", "cs_plan_create", "cs_plan_execute", "cs_query_batch",
              "cs_count_points", "cs_bitmap_build", "cs_plan_score", "cs_plan_compact", "cs_itemset_supports"):
        assert s in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol():
    from paper_1804_04640_b200 import _native

    lib = ctypes.CDLL(str(_native.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _native.SIGNATURES}
    assert bound == set(declared_symbols())


def test_no_device_fails_loudly():
    from paper_1804_04640_b200 import _native

    assert _native.lib.cs_abi_version() == 1
    n = ctypes.c_int32(-1)
    assert _native.lib.cs_device_count(ctypes.byref(n)) == 0
    if n.value == 0:
        h = ctypes.c_void_p()
        rc = _native.lib.cs_ctx_create(0, ctypes.byref(h))
        assert rc == _native.CS_ERR_CUDA
        assert b"no CUDA device" in _native.lib.cs_last_error()


def test_package_has_no_cpu_fallback():
    """The product package never imports the oracle."""
    pkg = ROOT / "paper_1804_04640_b200"
    for p in pkg.rglob("*.py"):
        src = p.read_text()
        assert not re.search(r"^\s*(import|from)\s+(oracle|gen_twin)\b", src, re.M), p
        assert "sys.path" not in src, p


def test_library_maps_on_first_call_not_at_import():
    """Importing the package (workload builders, query objects) does not map libcountgpu.so --
    bench.py's reference arm imports them and must run without the engine in the process --
    while the first call into the ABI does (and a missing library still fails at import)."""
    import subprocess
    import sys

    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_1804_04640_b200 as cs\n"
        "from paper_1804_04640_b200 import workloads, _native\n"
        "w = workloads.cfg1(nq=5)\n"
        "maps = lambda: 'libcountgpu' in open('/proc/self/maps').read()\n"
        "before = maps()\n"
        "_native.lib.cs_abi_version()\n"
        "print(before, maps(), _native.lib.loaded)\n" % str(ROOT)
    )
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout
    assert out.split() == ["False", "True", "True"]
