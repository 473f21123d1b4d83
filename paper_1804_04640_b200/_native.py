"""ctypes binding of libcountgpu.so (C ABI: include/countstream_gpu.h).

The engine has no CPU fallback: if the shared library is missing this module
raises at import time, and every call that fails on the device raises
:class:`EngineError` (or the reference's ``InvalidQueryError`` for bad queries).
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint32, c_uint64, c_void_p
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"
LIB_PATH = Path(os.environ.get("CS_LIB_PATH", LIB_DIR / "libcountgpu.so"))

CS_OK = 0
CS_ERR_INVALID = -1
CS_ERR_CUDA = -2
CS_ERR_OOM = -3
CS_ERR_UNSUPPORTED = -4
CS_ERR_PARSE = -5

CS_DELIM_SNIFF = -1
CS_DELIM_WHITESPACE = -2
CS_LOAD_OK, CS_LOAD_NO_RECORDS, CS_LOAD_BAD_RECORD, CS_LOAD_NEGATIVE = 0, 1, 2, 3
CS_LOAD_ARITY_COUNT, CS_LOAD_ARITY_SHORT, CS_LOAD_ARITY_ZERO = 4, 5, 6

CS_WANT_TABLES = 0x1
CS_WANT_LOGLIK = 0x2
CS_WANT_MI = 0x4
CS_WANT_NNZ = 0x8
CS_PARTIAL = 0x10
CS_NLOGN = 0x20

CS_REDUCE_ALLREDUCE = 0
CS_REDUCE_SCATTER = 1

# (name, restype, argtypes) for every symbol declared in include/countstream_gpu.h
_P = c_void_p
SIGNATURES = [
    ("cs_abi_version", c_int, []),
    ("cs_last_error", c_char_p, []),
    ("cs_device_count", c_int, [POINTER(c_int32)]),
    ("cs_ctx_create", c_int, [c_int32, POINTER(_P)]),
    ("cs_ctx_destroy", c_int, [_P]),
    ("cs_ctx_set_stream", c_int, [_P, _P]),
    ("cs_ctx_sync", c_int, [_P]),
    ("cs_ctx_launch_count", c_int, [_P, POINTER(c_int64)]),
    ("cs_ctx_last_kernel_ms", c_int, [_P, POINTER(ctypes.c_float)]),
    ("cs_ctx_itemset_class", c_int, [_P, POINTER(c_int32)]),
    ("cs_ctx_info", c_int, [_P, POINTER(c_int32), POINTER(c_int32), POINTER(c_int32)]),
    ("cs_db_create", c_int, [_P, _P, c_int32, c_int64, c_int64, _P, POINTER(_P)]),
    ("cs_db_create_empty", c_int, [_P, c_int32, c_int64, _P, POINTER(_P)]),
    ("cs_db_generate", c_int, [_P, c_int32, c_uint64, c_int64, c_int32, _P, _P, c_int64]),
    ("cs_db_destroy", c_int, [_P]),
    ("cs_db_shape", c_int, [_P, POINTER(c_int32), POINTER(c_int64), POINTER(c_int64)]),
    ("cs_db_columns", c_int, [_P, POINTER(_P), POINTER(c_int64)]),
    ("cs_db_download", c_int, [_P, c_int32, c_int64, c_int64, _P]),
    ("cs_db_set_total_rows", c_int, [_P, c_int64]),
    ("cs_db_arities", c_int, [_P, _P]),
    ("cs_db_load_text", c_int, [_P, _P, c_int64, c_int32, _P, c_int32, POINTER(_P), _P]),
    ("cs_bitmap_build", c_int, [_P, c_int32, _P]),
    ("cs_bitmap_plane", c_int, [_P, c_int32, c_int32, POINTER(_P), POINTER(c_int64)]),
    ("cs_plan_create", c_int, [_P, c_int32, _P, _P, c_uint32, POINTER(_P)]),
    ("cs_plan_info", c_int, [_P, _P, _P, POINTER(c_int64)]),
    ("cs_plan_execute", c_int, [_P, _P, _P, _P, _P]),
    ("cs_plan_score", c_int, [_P, _P, _P, _P, _P]),
    ("cs_plan_compact", c_int, [_P, _P, _P, c_int64, _P, _P, _P]),
    ("cs_plan_destroy", c_int, [_P]),
    ("cs_family_scores", c_int, [_P, c_int64, _P, c_int64, _P, _P, _P, c_double, _P, _P]),
    ("cs_query_batch", c_int, [_P, c_int32, _P, _P, c_uint32, _P, _P, _P, _P]),
    ("cs_query_one", c_int, [_P, c_int32, _P, c_uint32, _P, _P, _P, _P]),
    ("cs_query_one_cells", c_int, [_P, c_int32, _P, _P, _P, _P, _P]),
    ("cs_comm_unique_id", c_int, [_P]),
    ("cs_comm_init", c_int, [_P, _P, c_int32, c_int32]),
    ("cs_comm_destroy", c_int, [_P]),
    ("cs_reduce_tables", c_int, [_P, _P, c_int64, c_int32, _P]),
    ("cs_comm_all_gather", c_int, [_P, _P, c_int64, _P]),
    ("cs_count_points", c_int, [_P, c_int32, _P, _P, _P, _P]),
    ("cs_itemset_supports", c_int, [_P, c_int32, _P, _P, _P]),
]


class EngineError(RuntimeError):
    """A device-side failure reported by libcountgpu."""

    def __init__(self, code: int, message: str):
        super().__init__(f"libcountgpu error {code}: {message}")
        self.code = code


def _require() -> None:
    if not LIB_PATH.exists():
        raise ImportError(
            f"libcountgpu.so not found at {LIB_PATH}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)"
        )


def _load() -> ctypes.CDLL:
    _require()
    lib = ctypes.CDLL(str(LIB_PATH))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.cs_abi_version() != 1:  # pragma: no cover - build skew
        raise ImportError(f"libcountgpu ABI {lib.cs_abi_version()} != 1")
    return lib


class _LazyLib:
    """The library handle, mapped into the process on the first call into it (not at import):
    importing the package for its host-side pieces (workload builders, query objects -- e.g.
    bench.py's reference arm) does not load the engine.  A missing library still fails at
    import (the check below), and every call goes to the CUDA engine: there is no fallback."""

    _lib: ctypes.CDLL | None = None

    def _get(self) -> ctypes.CDLL:
        if _LazyLib._lib is None:
            _LazyLib._lib = _load()
        return _LazyLib._lib

    @property
    def loaded(self) -> bool:
        return _LazyLib._lib is not None

    def __getattr__(self, name):
        return getattr(self._get(), name)


_require()
lib = _LazyLib()


def check(rc: int) -> None:
    """Raise on a non-zero return code, mapping CS_ERR_INVALID to InvalidQueryError."""
    if rc == CS_OK:
        return
    msg = (lib.cs_last_error() or b"").decode(errors="replace")
    if rc == CS_ERR_INVALID:
        from .database import InvalidQueryError

        raise InvalidQueryError(msg)
    if rc == CS_ERR_UNSUPPORTED:
        from .database import UnsupportedQueryError

        raise UnsupportedQueryError(msg)
    raise EngineError(rc, msg)


def last_error() -> str:
    return (lib.cs_last_error() or b"").decode(errors="replace")


def ptr(x) -> int | None:
    """Address of a numpy array or torch tensor (None passes NULL)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    return x.ctypes.data


def device_count() -> int:
    n = c_int32(0)
    check(lib.cs_device_count(ctypes.byref(n)))
    return int(n.value)
