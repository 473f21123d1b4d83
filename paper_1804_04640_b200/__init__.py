"""countstream on B200: batched counting queries on sm_100a (arXiv 1804.04640 hot path).

Drop-in for the reference package ``countstream``'s counting API: the same
``Database`` / ``QuerySpec`` / ``Assignment`` descriptors, the same
``(N_ijk, N_ij)`` aggregator protocol and the same ``Strategy`` facade, with
the counting done by hand-written CUDA kernels behind the C ABI of
``lib/libcountgpu.so`` (include/countstream_gpu.h).  Importing the package
loads that library; there is no CPU fallback.
"""

from .aggregators import (
    Aggregator,
    AggregatorContractError,
    LogLikelihood,
    MdlScore,
    MutualInformation,
    NullSink,
    Record,
    RecordCollector,
    mdl_score,
)
from .database import (
    Assignment,
    Database,
    DatabaseLoadError,
    InvalidQueryError,
    QuerySpec,
    UnsupportedQueryError,
    generate_synthetic,
    load_arities,
    load_csv,
    parse_synthetic,
)
from .engine import GpuContext, GpuDatabase, QueryPlan, encode_queries
from .harness import (
    STRATEGY_NAMES,
    AssociationRule,
    BenchResult,
    DeviceDatabase,
    GpuStrategy,
    ParentSetResult,
    RandomQueryStream,
    Strategy,
    bench_random,
    learn_parents,
    load_csv_device,
    make_strategies,
    mine_rules,
    shared_context,
)
from ._native import EngineError, LIB_PATH

__version__ = "0.1.0"

__all__ = [
    "Aggregator",
    "AggregatorContractError",
    "LogLikelihood",
    "MdlScore",
    "MutualInformation",
    "NullSink",
    "Record",
    "RecordCollector",
    "mdl_score",
    "Assignment",
    "Database",
    "DatabaseLoadError",
    "InvalidQueryError",
    "QuerySpec",
    "UnsupportedQueryError",
    "generate_synthetic",
    "load_arities",
    "load_csv",
    "parse_synthetic",
    "GpuContext",
    "GpuDatabase",
    "QueryPlan",
    "encode_queries",
    "STRATEGY_NAMES",
    "AssociationRule",
    "BenchResult",
    "DeviceDatabase",
    "GpuStrategy",
    "ParentSetResult",
    "RandomQueryStream",
    "Strategy",
    "bench_random",
    "learn_parents",
    "load_csv_device",
    "make_strategies",
    "mine_rules",
    "shared_context",
    "EngineError",
    "LIB_PATH",
]
