"""B200-native single-pass sufficient-statistics engine (n, column sums, packed X^T X).

Drop-in for the reference's dataset_suffstats / accumulate_chunk path; see DESIGN.md.
"""
from .sstat import (  # noqa: F401
    Chunk,
    CoMoments,
    ColumnSumResult,
    DatasetSchema,
    DeviceError,
    Engine,
    Error,
    FormatError,
    IoError,
    NonFiniteError,
    Partition,
    PrecisionMode,
    ReductionError,
    ReductionPlan,
    ReductionTimings,
    RowRange,
    RowReader,
    SchemaMismatchError,
    SuffStats,
    accumulate_chunk,
    dataset_suffstats,
    default_engine,
    fold_range_partials,
    merge_suffstats,
    packed_index,
    plan_partitions,
    shard_ranges,
)
from . import _native  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
