"""ctypes binding of libsstat_b200.so (the C ABI declared in include/sstat_cuda.h).

The library is the product: there is no Python or CPU fallback for the hot path.
Loading fails loudly (NativeLibraryError) when the shared object is missing; build it
with ``python -c "import __graft_entry__ as g; g.build()"`` or ``make -C
paper_2604_23826_b200/csrc``.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_char, c_char_p, c_double, c_int, c_size_t, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSTAT_LIB", os.path.join(HERE, "libsstat_b200.so"))

# sstat_status
OK = 0
ERR_NONFINITE = 1
ERR_SCHEMA = 2
ERR_INVALID = 3
ERR_CUDA = 4
ERR_NCCL = 5
ERR_OOM = 6
ERR_UNSUPPORTED = 7
ERR_IO = 8
ERR_FORMAT = 9
ERR_PEER = 10

SRC_DEVICE = 0
SRC_HOST = 1
SRC_FILE = 2
SRC_READER = 3

FLAG_NO_SHIFT = 1 << 0
FLAG_REFEXACT = 1 << 1

GEN_MIXED = 0
GEN_ID_GAUSS = 1
GEN_GAUSS = 2

# Exported symbols, one per declaration in include/sstat_cuda.h (checked by tests).
EXPORTS = (
    "sstat_cuda_abi_version",
    "sstat_status_string",
    "sstat_cuda_init",
    "sstat_cuda_init_devices",
    "sstat_cuda_device_count",
    "sstat_cuda_destroy",
    "sstat_cuda_set_stream",
    "sstat_cuda_set_staging",
    "sstat_cuda_set_host_threads",
    "sstat_cuda_nccl_unique_id",
    "sstat_cuda_comm_init",
    "sstat_shard_ranges",
    "sstat_cuda_accumulate",
    "sstat_cuda_dataset",
    "sstat_cuda_range_partials",
    "sstat_cuda_column_sum",
    "sstat_cuda_comoments",
    "sstat_fold_ranges_host",
    "sstat_plan_partitions",
    "sstat_merge",
    "sstat_cuda_generate",
)


class NativeLibraryError(RuntimeError):
    """libsstat_b200.so is missing or unusable: the CUDA path cannot run."""


class Error(Structure):
    _fields_ = [
        ("row", c_uint64),
        ("col", c_uint32),
        ("status", c_uint32),
        ("range_index", c_uint64),
        ("msg", c_char * 256),
    ]


class Timings(Structure):
    _fields_ = [
        ("h2d_seconds", c_double),
        ("kernel_seconds", c_double),
        ("exchange_seconds", c_double),
        ("fold_seconds", c_double),
        ("total_seconds", c_double),
        ("bytes_read", c_uint64),
        ("h2d_bytes", c_uint64),
        ("kernel_launches", c_uint32),
        ("n_local_ranges", c_uint32),
        ("kernel", c_char * 96),
    ]


# sstat_read_rows_fn: (user, first_row, n_rows, scratch) -> rows pointer (NULL = failure)
READ_ROWS_FN = ctypes.CFUNCTYPE(c_void_p, c_void_p, c_uint64, c_uint64, c_void_p)


class Source(Structure):
    _fields_ = [
        ("kind", c_uint32),
        ("reserved", c_uint32),
        ("ptr", c_void_p),
        ("first_row", c_uint64),
        ("n_rows", c_uint64),
        ("path", c_char_p),
        ("read_rows", READ_ROWS_FN),
        ("user", c_void_p),
    ]


class ColumnSum(Structure):
    _fields_ = [
        ("float_sum", c_double),
        ("exact_ok", c_int),
        ("float_matches_exact", c_int),
        ("exact_hi", ctypes.c_int64),
        ("exact_lo", c_uint64),
        ("note_row", c_uint64),
    ]


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and prototype the C ABI."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not found: the B200 CUDA engine is not built (run __graft_entry__.build())"
        )
    try:
        lib = ctypes.CDLL(path)
    except OSError as e:  # pragma: no cover - depends on the host
        raise NativeLibraryError(f"cannot load {path}: {e}") from e
    P = POINTER
    u64p, dp = P(c_uint64), P(c_double)
    proto = {
        "sstat_cuda_abi_version": (c_int, []),
        "sstat_status_string": (c_char_p, [c_int]),
        "sstat_cuda_init": (c_int, [P(c_void_p), c_int]),
        "sstat_cuda_init_devices": (c_int, [P(c_void_p), c_int, P(c_int)]),
        "sstat_cuda_device_count": (c_int, [c_void_p]),
        "sstat_cuda_destroy": (c_int, [c_void_p]),
        "sstat_cuda_set_stream": (c_int, [c_void_p, c_void_p]),
        "sstat_cuda_set_staging": (c_int, [c_void_p, c_uint32, c_uint64]),
        "sstat_cuda_set_host_threads": (c_int, [c_void_p, c_uint32]),
        "sstat_cuda_nccl_unique_id": (c_int, [c_void_p, c_size_t]),
        "sstat_cuda_comm_init": (c_int, [c_void_p, c_int, c_int, c_void_p, c_size_t]),
        "sstat_shard_ranges": (c_int, [c_uint64, c_int, c_int, u64p, u64p]),
        "sstat_cuda_accumulate": (
            c_int,
            [c_void_p, c_void_p, c_uint64, c_uint32, c_uint64, c_uint32, c_uint32, u64p, dp, dp, P(Error)],
        ),
        "sstat_cuda_dataset": (  # sums_out / cross_out as addresses (the hot call passes ints)
            c_int,
            [c_void_p, P(Source), c_uint32, c_void_p, c_void_p, c_uint64, c_uint32, c_uint32, u64p, c_void_p,
             c_void_p, P(Timings), P(Error)],
        ),
        "sstat_cuda_range_partials": (
            c_int,
            [c_void_p, P(Source), c_uint32, c_void_p, c_void_p, c_uint64, c_uint64, c_uint64, c_uint32, c_uint32, dp,
             P(Error)],
        ),
        "sstat_cuda_column_sum": (
            c_int,
            [c_void_p, P(Source), c_uint32, c_uint32, c_void_p, c_void_p, c_uint64, c_uint32, c_uint32, P(ColumnSum),
             P(Error)],
        ),
        "sstat_cuda_comoments": (
            c_int, [c_void_p, P(Source), c_uint32, c_void_p, c_void_p, c_uint64, c_uint32, u64p, dp, dp, P(Error)]
        ),
        "sstat_fold_ranges_host": (c_int, [dp, c_uint64, c_uint64, c_int, c_uint32, c_uint32, c_uint32, dp]),
        "sstat_plan_partitions": (c_uint64, [c_uint64, c_uint64, c_void_p, c_void_p]),
        "sstat_merge": (c_int, [c_uint32, c_uint32, u64p, dp, dp, c_uint64, dp, dp]),
        "sstat_cuda_generate": (
            c_int, [c_void_p, c_void_p, c_uint32, c_uint64, c_double, c_uint32, c_uint64, c_uint64, c_uint32]
        ),
    }
    for name, (res, args) in proto.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def status_string(code: int) -> str:
    return load().sstat_status_string(code).decode()
