"""Host-side mirror of the reference's sufficient-statistics interface, over the B200 engine.

Names, argument meaning and error behaviour follow the reference
(paths relative to /root/reference/proj):

  DatasetSchema                   include/sstat/schema.hpp:15-62
  PrecisionMode, RowRange,
  Partition, ReductionPlan,
  ReductionTimings                include/sstat/reduce.hpp:18-60
  plan_partitions                 src/reduce.cpp:8-16
  Chunk                           include/sstat/chunk.hpp:13-24
  SuffStats                       include/sstat/suffstats.hpp:19-30 (cross = SymPacked,
                                  include/sstat/linalg.hpp:50-81)
  accumulate_chunk                src/suffstats.cpp:74-84
  merge_suffstats                 src/suffstats.cpp:86-105
  dataset_suffstats               src/suffstats.cpp:279-288 (run_reduction,
                                  include/sstat/reduce.hpp:70-146)
  Error hierarchy                 include/sstat/errors.hpp:12-94

Every accumulation runs on the GPU through libsstat_b200.so (the C ABI of
include/sstat_cuda.h).  There is no CPU fallback: without the library or a CUDA
device the calls raise.
"""
from __future__ import annotations

import ctypes
import enum
import os
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N


# ---------------------------------------------------------------- errors (errors.hpp)
class Error(RuntimeError):
    """Base class for all engine errors (errors.hpp:12-16)."""


class IoError(Error):
    pass


class FormatError(Error):
    pass


class SchemaMismatchError(Error):
    pass


class NonFiniteError(Error):
    """Non-finite value; row absolute 0-based, column 0-based (errors.hpp:59-72)."""

    def __init__(self, row: int, column: int, what: str):
        super().__init__(what)
        self._row, self._column = row, column

    def row(self) -> int:
        return self._row

    def column(self) -> int:
        return self._column


class ReductionError(Error):
    """A per-chunk job failed inside a reduction (errors.hpp:85-92)."""

    def __init__(self, range_index: int, what: str, cause: Optional[Error] = None):
        super().__init__(what)
        self._range_index = range_index
        self.cause = cause

    def range_index(self) -> int:
        return self._range_index


class DeviceError(Error):
    """CUDA / NCCL / out-of-memory / unsupported: no reference equivalent."""

    def __init__(self, status: int, what: str):
        super().__init__(what)
        self.status = status


# ---------------------------------------------------------------- plan types (reduce.hpp)
class PrecisionMode(enum.IntEnum):
    Binary64 = 0
    Binary32Diagnostic = 1


@dataclass(frozen=True)
class RowRange:
    start_row: int = 0
    row_count: int = 0


class _RangeList(list):
    """A list of RowRange that counts its own mutations: the key of Partition's cached C-ABI
    arrays, so any in-place change (item assignment, append, sort, ...) rebuilds them while an
    unchanged plan costs O(1) per call.  RowRange is frozen, so elements cannot change in place."""

    __slots__ = ("version",)

    def __init__(self, items=()):
        super().__init__(items)
        self.version = 0


def _counting(name):
    base = getattr(list, name)

    def method(self, *args, **kwargs):
        self.version += 1
        return base(self, *args, **kwargs)

    method.__name__ = name
    return method


for _name in ("__setitem__", "__delitem__", "__iadd__", "__imul__", "append", "extend", "insert", "pop", "remove",
              "clear", "sort", "reverse"):
    setattr(_RangeList, _name, _counting(_name))


@dataclass
class Partition:
    ranges: List[RowRange] = field(default_factory=list)

    def __setattr__(self, name, value):
        if name == "ranges" and not isinstance(value, _RangeList):
            value = _RangeList(value)
        object.__setattr__(self, name, value)

    def total_rows(self) -> int:
        return sum(r.row_count for r in self.ranges)

    def arrays(self):
        """(starts, counts) as uint64 arrays for the C ABI, cached while the ranges are unchanged."""
        return self._cached()[1:3]

    def addresses(self):
        """(starts address, counts address, n) of the cached arrays (the hot call's arguments)."""
        return self._cached()[3]

    def _cached(self):
        key = (id(self.ranges), self.ranges.version, len(self.ranges))
        cached = getattr(self, "_arrays", None)
        if cached is None or cached[0] != key:
            starts = np.fromiter((r.start_row for r in self.ranges), dtype=np.uint64, count=len(self.ranges))
            counts = np.fromiter((r.row_count for r in self.ranges), dtype=np.uint64, count=len(self.ranges))
            cached = (key, starts, counts, (starts.ctypes.data, counts.ctypes.data, len(self.ranges)))
            self._arrays = cached
        return cached


@dataclass
class ReductionPlan:
    partition: Partition = field(default_factory=Partition)
    worker_count: int = 1  # accepted for API parity; the device decides its own parallelism
    precision: PrecisionMode = PrecisionMode.Binary64


@dataclass
class ReductionTimings:
    read_seconds: float = 0.0  # host->device copy time (streamed sources)
    work_seconds: float = 0.0  # accumulate + fold kernels (device events)
    bytes_read: int = 0
    exchange_seconds: float = 0.0
    total_seconds: float = 0.0
    kernel_launches: int = 0


def plan_partitions(n_rows: int, chunk_rows: int) -> Partition:
    """ceil(n_rows / chunk_rows) ranges (reduce.cpp:8-16); invalid_argument on 0."""
    if chunk_rows == 0:
        raise ValueError("plan_partitions: chunk_rows must be >= 1")
    if n_rows == 0:
        raise ValueError("plan_partitions: n_rows must be >= 1")
    return Partition([RowRange(s, min(chunk_rows, n_rows - s)) for s in range(0, n_rows, chunk_rows)])


# ---------------------------------------------------------------- schema / stats
@dataclass
class DatasetSchema:
    column_names: List[str] = field(default_factory=list)
    identifier_columns: List[int] = field(default_factory=list)

    def column_count(self) -> int:
        return len(self.column_names)

    def is_identifier(self, column: int) -> bool:
        return column in self.identifier_columns

    def validate(self) -> None:
        if not self.column_names:
            raise ValueError("schema: column count must be >= 1")
        prev = -1
        for c in self.identifier_columns:
            if c >= len(self.column_names):
                raise ValueError("schema: identifier column out of range")
            if c <= prev:
                raise ValueError("schema: identifier columns must be sorted and unique")
            prev = c

    @staticmethod
    def table1() -> "DatasetSchema":
        return DatasetSchema(list("ABCDEFGHIJK"), [0])

    @staticmethod
    def iid_uniform(p: int) -> "DatasetSchema":
        return DatasetSchema(["A"] + [f"U{i}" for i in range(1, p + 1)], [0])

    @staticmethod
    def generic(p: int, leading_identifier: bool = True) -> "DatasetSchema":
        return DatasetSchema([f"c{i}" for i in range(1, p + 1)], [0] if leading_identifier and p > 0 else [])


def packed_index(p: int, j: int, k: int) -> int:
    if j > k:
        j, k = k, j
    return j * p - j * (j - 1) // 2 + (k - j)


@dataclass
class SuffStats:
    n: int
    sums: np.ndarray  # [p] float64
    cross: np.ndarray  # [p(p+1)/2] float64, SymPacked order
    schema: DatasetSchema
    precision: PrecisionMode = PrecisionMode.Binary64

    @staticmethod
    def empty(schema: DatasetSchema, precision: PrecisionMode = PrecisionMode.Binary64) -> "SuffStats":
        schema.validate()
        p = schema.column_count()
        return SuffStats(0, np.zeros(p), np.zeros(p * (p + 1) // 2), schema, PrecisionMode(precision))

    def cross_at(self, j: int, k: int) -> float:
        return float(self.cross[packed_index(len(self.sums), j, k)])

    def cross_full(self) -> np.ndarray:
        p = len(self.sums)
        m = np.zeros((p, p))
        iu = np.triu_indices(p)
        m[iu] = self.cross
        m[(iu[1], iu[0])] = self.cross
        return m

    def __eq__(self, other: object) -> bool:  # the defaulted operator== (value equality)
        if not isinstance(other, SuffStats):
            return NotImplemented
        return (
            self.n == other.n
            and self.schema == other.schema
            and self.precision == other.precision
            and np.array_equal(self.sums, other.sums)
            and np.array_equal(self.cross, other.cross)
        )

    def bit_equal(self, other: "SuffStats") -> bool:
        return (
            self.n == other.n
            and np.array_equal(self.sums.view(np.uint64), other.sums.view(np.uint64))
            and np.array_equal(self.cross.view(np.uint64), other.cross.view(np.uint64))
        )


@dataclass
class ColumnSumResult:
    """ColumnSumResult (reduce.hpp:148-158)."""

    float_sum: float
    exact_sum: Optional[int]
    float_matches_exact: bool
    exact_note: Optional[str]


@dataclass
class CoMoments:
    """Centered co-moments (suffstats.hpp:35-45): n, mean, M2 packed."""

    n: int
    mean: np.ndarray
    m2: np.ndarray
    schema: DatasetSchema


@dataclass
class Chunk:
    """Row-major block of rows (chunk.hpp:13-24); values: numpy array or torch tensor."""

    start_row: int
    row_count: int
    column_count: int
    values: object


def merge_suffstats(a: SuffStats, b: SuffStats) -> SuffStats:
    """Elementwise merge (suffstats.cpp:86-105) via the library's host merge."""
    if a.schema != b.schema:
        raise SchemaMismatchError("merge_suffstats: schemas differ")
    if a.precision != b.precision:
        raise SchemaMismatchError("merge_suffstats: precision modes differ")
    lib = N.load()
    n = ctypes.c_uint64(a.n)
    sums = np.ascontiguousarray(a.sums, dtype=np.float64).copy()
    cross = np.ascontiguousarray(a.cross, dtype=np.float64).copy()
    bs = np.ascontiguousarray(b.sums, dtype=np.float64)
    bc = np.ascontiguousarray(b.cross, dtype=np.float64)
    dp = ctypes.POINTER(ctypes.c_double)
    st = lib.sstat_merge(len(sums), int(a.precision), ctypes.byref(n), sums.ctypes.data_as(dp), cross.ctypes.data_as(dp),
                         b.n, bs.ctypes.data_as(dp), bc.ctypes.data_as(dp))
    if st != N.OK:
        raise ValueError(N.status_string(st))
    return SuffStats(n.value, sums, cross, a.schema, a.precision)


# ---------------------------------------------------------------- the engine
def _raise(status: int, err: N.Error, in_dataset: bool, reader=None) -> None:
    msg = err.msg.decode(errors="replace")
    if status == N.ERR_IO and isinstance(reader, RowReader) and reader.error is not None:
        raise IoError(f"{msg}: {reader.error!r}") from reader.error
    if status == N.ERR_NONFINITE:
        nf = NonFiniteError(err.row, err.col, f"non-finite value at row {err.row}, column {err.col}")
        if in_dataset:
            raise ReductionError(err.range_index, msg, nf)
        raise nf
    if status == N.ERR_SCHEMA:
        if in_dataset and msg.startswith("range "):
            raise ReductionError(err.range_index, msg, SchemaMismatchError(msg))
        raise SchemaMismatchError(msg)
    if status == N.ERR_INVALID:
        raise ValueError(msg)
    if status == N.ERR_IO:
        raise IoError(msg)
    if status == N.ERR_FORMAT:
        raise FormatError(msg)
    raise DeviceError(status, f"{N.status_string(status)}: {msg}")


def _is_torch_cuda(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _current_raw_stream(tensor) -> int:
    """torch's current cudaStream_t on the tensor's device (the raw getter: ~0.1 us instead of
    ~2 us for a torch.cuda.Stream object)."""
    import torch

    get = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if get is not None:
        return int(get(tensor.device.index))
    return torch.cuda.current_stream(tensor.device).cuda_stream


class RowReader:
    """A dataset served by a callback: BinaryReader::read_rows (binfile.cpp:140-161) as the C
    ABI's SSTAT_SRC_READER.  ``read(first_row, n_rows, scratch) -> address`` either fills the
    pinned ``scratch`` buffer (n_rows * p * 8 bytes at that address) and returns it, or returns
    the address of host memory already holding the rows (pinned memory goes to the device by
    DMA directly), valid until the pass returns; 0 / None = read failure.  ``n_rows`` = the
    dataset's rows.  The engine calls it once per staging slot (256 MiB by default)."""

    def __init__(self, read, n_rows: int, first_row: int = 0):
        self.n_rows, self.first_row = int(n_rows), int(first_row)
        self.error: Optional[BaseException] = None

        def trampoline(_user, row, n, scratch):
            try:
                return int(read(row, n, scratch) or 0) or None
            except BaseException as e:  # surfaced as IoError by the engine's NULL path
                self.error = e
                return None

        self._fn = N.READ_ROWS_FN(trampoline)  # kept alive with the reader


class Engine:
    """One context of the B200 engine (sstat_cuda_ctx): one device, or with ``devices`` a
    device group — one process driving several GPUs (sstat_cuda_init_devices)."""

    def __init__(self, device: Optional[int] = None, devices: Optional[Sequence[int]] = None):
        self._lib = N.load()
        self._ctx = ctypes.c_void_p()
        if devices is not None:
            devs = [int(d) for d in devices]
            arr = (ctypes.c_int * len(devs))(*devs)
            st = self._lib.sstat_cuda_init_devices(ctypes.byref(self._ctx), len(devs), arr)
            if st != N.OK:
                raise DeviceError(st, f"sstat_cuda_init_devices failed: {N.status_string(st)}")
            self.devices = devs
            self._group = True
        else:
            st = self._lib.sstat_cuda_init(ctypes.byref(self._ctx), -1 if device is None else int(device))
            if st != N.OK:
                raise DeviceError(st, f"sstat_cuda_init failed: {N.status_string(st)}")
            self.devices = [device]
            self._group = False
        self.rank, self.world = 0, 1
        self._stream_explicit = False  # set_stream called: never re-bind
        self._stream_bound = None  # the torch stream handle the context currently launches on
        # dataset_suffstats fills last_timings (device events around the kernels) when this is True
        # or a ReductionTimings is passed — like the reference, timings cost nothing unless asked
        # for: each device event costs ~5-7 us of a call (C1: 43 us untimed, 65 us timed)
        self.collect_timings = False
        self.last_timings = None

    @property
    def n_devices(self) -> int:
        return len(self.devices)

    def close(self) -> None:
        if self._ctx:
            self._lib.sstat_cuda_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # -- configuration
    def set_stream(self, cuda_stream: int) -> None:
        """Launch on an external cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream).
        Without this call, a CUDA-tensor source binds the context to torch's current stream of
        the tensor's device, so the pass is ordered after whatever produced the tensor."""
        self._check(self._lib.sstat_cuda_set_stream(self._ctx, ctypes.c_void_p(cuda_stream or None)))
        self._stream_explicit = True
        self._stream_bound = cuda_stream

    @staticmethod
    def _wait_producer(tensor) -> None:
        """A group member launches on its own blocking stream, ordered after the legacy default
        stream only: a shard produced on another torch stream is waited for on the host first."""
        if _current_raw_stream(tensor) != 0:
            import torch

            torch.cuda.current_stream(tensor.device).synchronize()

    def _follow_torch_stream(self, tensor) -> None:
        if self._stream_explicit or self._group:
            return  # group members keep their own (blocking) streams
        h = _current_raw_stream(tensor)
        if h != self._stream_bound:
            self._check(self._lib.sstat_cuda_set_stream(self._ctx, ctypes.c_void_p(h or None)))
            self._stream_bound = h

    def set_staging(self, slots: int, slot_bytes: int) -> None:
        self._check(self._lib.sstat_cuda_set_staging(self._ctx, slots, slot_bytes))

    def set_host_threads(self, threads: int) -> None:
        """Feeder threads for pageable-host and file sources (0 = default); results unchanged."""
        self._check(self._lib.sstat_cuda_set_host_threads(self._ctx, threads))

    def init_distributed(self, rank: int, world: int, unique_id: Optional[bytes]) -> None:
        """Attach an NCCL communicator (one process per GPU)."""
        buf = ctypes.create_string_buffer(unique_id, 128) if unique_id is not None else None
        self._check(self._lib.sstat_cuda_comm_init(self._ctx, rank, world, buf, 128 if buf is not None else 0))
        self.rank, self.world = rank, world

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = N.load()
        buf = ctypes.create_string_buffer(128)
        st = lib.sstat_cuda_nccl_unique_id(buf, 128)
        if st != N.OK:
            raise DeviceError(st, "ncclGetUniqueId failed")
        return buf.raw

    def _check(self, st: int) -> None:
        if st != N.OK:
            raise DeviceError(st, N.status_string(st))

    # -- hot path
    def accumulate_chunk(self, chunk: Chunk, schema: DatasetSchema,
                         precision: PrecisionMode = PrecisionMode.Binary64, flags: int = 0) -> SuffStats:
        """accumulate_chunk (suffstats.cpp:74-84) on a host or device chunk."""
        schema.validate()
        p = schema.column_count()
        if chunk.column_count != p:
            raise SchemaMismatchError(f"chunk has {chunk.column_count} columns, schema has {p}")
        ptr, keep = self._rows_pointer(chunk.values, chunk.row_count * p)
        out = SuffStats.empty(schema, precision)
        n = ctypes.c_uint64()
        err = N.Error()
        dp = ctypes.POINTER(ctypes.c_double)
        st = self._lib.sstat_cuda_accumulate(self._ctx, ptr, chunk.row_count, p, chunk.start_row, int(precision), flags,
                                             ctypes.byref(n), out.sums.ctypes.data_as(dp),
                                             out.cross.ctypes.data_as(dp), ctypes.byref(err))
        del keep
        if st != N.OK:
            _raise(st, err, in_dataset=False)
        out.n = n.value
        return out

    def dataset_suffstats(self, dataset, schema: DatasetSchema, plan: ReductionPlan,
                          timings: Optional[ReductionTimings] = None, flags: int = 0,
                          first_row: int = 0, n_rows: Optional[int] = None) -> SuffStats:
        """dataset_suffstats (suffstats.cpp:279-288).

        dataset: an SSTATBIN path, a CUDA tensor (HBM-resident rows), a host array
        (numpy / CPU tensor; pinned memory is copied by DMA) or a RowReader.  With a
        communicator, each rank passes its shard and ``first_row`` = the absolute index of its
        row 0.  A device group takes a path / host array / reader (every member reads its own
        ranges) or a list of CUDA tensors, one shard per member in device order (the shard rule
        of shard_ranges; first rows follow from the plan).
        """
        schema.validate()
        p = schema.column_count()
        src, keep = self._source(dataset, p, first_row, n_rows, plan)
        a_starts, a_counts, R = plan.partition.addresses()
        # one ctypes buffer [sums | cross] viewed by numpy: no per-call pointer objects
        E = p + p * (p + 1) // 2
        res = (ctypes.c_double * E)()
        a_res = ctypes.addressof(res)
        n = ctypes.c_uint64()
        err = N.Error()
        tm = N.Timings() if (timings is not None or self.collect_timings) else None
        st = self._lib.sstat_cuda_dataset(self._ctx, src, p, a_starts, a_counts, R,
                                          int(plan.precision), flags, ctypes.byref(n), a_res, a_res + 8 * p,
                                          ctypes.byref(tm) if tm is not None else None, ctypes.byref(err))
        if st != N.OK:
            _raise(st, err, in_dataset=True, reader=dataset)
        del keep
        flat = np.frombuffer(res, dtype=np.float64)
        out = SuffStats(n.value, flat[:p], flat[p:], schema, PrecisionMode(plan.precision))
        if timings is not None and tm is not None:
            timings.read_seconds = tm.h2d_seconds
            timings.work_seconds = tm.kernel_seconds + tm.fold_seconds
            timings.bytes_read = tm.bytes_read
            timings.exchange_seconds = tm.exchange_seconds
            timings.total_seconds = tm.total_seconds
            timings.kernel_launches = tm.kernel_launches
        self.last_timings = tm
        return out

    def range_partials(self, dataset, schema: DatasetSchema, plan: ReductionPlan, first_range: int,
                       last_range: int, flags: int = 0, first_row: int = 0,
                       n_rows: Optional[int] = None) -> np.ndarray:
        """Per-range partials [sums | packed cross] of ranges [first_range, last_range) in raw space,
        without the fold: what a rank contributes to the exchange, or a checkpoint of finished
        ranges (run_reduction's partials slots, reduce.hpp:85,108).  Shape (last - first, E)."""
        schema.validate()
        p = schema.column_count()
        src, keep = self._source(dataset, p, first_row, n_rows, plan)
        starts, counts = plan.partition.arrays()
        E = p + p * (p + 1) // 2
        out = np.zeros((max(last_range - first_range, 0), E))
        err = N.Error()
        st = self._lib.sstat_cuda_range_partials(self._ctx, src, p, starts.ctypes.data,
                                                 counts.ctypes.data, len(starts), first_range, last_range,
                                                 int(plan.precision), flags,
                                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(err))
        del keep
        if st != N.OK:
            _raise(st, err, in_dataset=True)
        return out

    def _source(self, dataset, p: int, first_row: int, n_rows: Optional[int], plan: Optional[ReductionPlan] = None):
        """(pointer to sstat_cuda_source[k], objects to keep alive) for a call's dataset."""
        if isinstance(dataset, (list, tuple)):  # a device group's per-member shards
            if len(dataset) != self.n_devices or plan is None:
                raise ValueError(f"expected one CUDA shard per device ({self.n_devices}), got {len(dataset)}")
            R = len(plan.partition.ranges)
            srcs = (N.Source * len(dataset))()
            keep = []
            for i, shard in enumerate(dataset):
                if not _is_torch_cuda(shard):
                    raise TypeError("device-group shards must be CUDA tensors")
                self._wait_producer(shard)
                f, _ = shard_ranges(R, i, len(dataset))
                _check_width(shard, p)
                ptr, k = self._rows_pointer(shard, None)
                keep.append(k)
                srcs[i].kind = N.SRC_DEVICE
                srcs[i].ptr = ptr
                srcs[i].first_row = plan.partition.ranges[f].start_row if f < R else 0
                srcs[i].n_rows = _rows_of(shard, p)
            return srcs, (srcs, keep)
        src = N.Source()
        if type(dataset).__module__.startswith("torch") and getattr(dataset, "is_cuda", False):
            # the common HBM-resident case, without the generic helpers' repeated type probes
            shape = dataset.shape
            if len(shape) >= 2 and shape[-1] != p or len(shape) < 2:
                _check_width(dataset, p)
            ptr, keep = self._rows_pointer(dataset, None)
            if self._group:
                self._wait_producer(dataset)
            else:
                self._follow_torch_stream(dataset)
            src.kind = N.SRC_DEVICE
            src.ptr = ptr
            src.first_row = first_row
            src.n_rows = n_rows if n_rows is not None else dataset.numel() // p
            return ctypes.pointer(src), (src, keep)
        if isinstance(dataset, (str, os.PathLike)):
            keep = os.fsencode(os.fspath(dataset))
            src.kind = N.SRC_FILE
            src.path = keep
        elif isinstance(dataset, RowReader):
            keep = dataset
            dataset.error = None
            src.kind = N.SRC_READER
            src.read_rows = dataset._fn
            src.first_row = dataset.first_row
            src.n_rows = dataset.n_rows
        else:
            _check_width(dataset, p)
            ptr, keep = self._rows_pointer(dataset, None)
            cuda = _is_torch_cuda(dataset)
            if cuda and self._group:
                self._wait_producer(dataset)
            elif cuda:
                self._follow_torch_stream(dataset)
            src.kind = N.SRC_DEVICE if cuda else N.SRC_HOST
            src.ptr = ptr
            src.first_row = first_row
            src.n_rows = n_rows if n_rows is not None else _rows_of(dataset, p)
        return ctypes.pointer(src), (src, keep)

    def column_sum(self, dataset, column: int, plan: ReductionPlan, p: Optional[int] = None, flags: int = 0,
                   first_row: int = 0, n_rows: Optional[int] = None) -> ColumnSumResult:
        """column_sum (reduce.cpp:32-88); p = the dataset's column count (files: from the header)."""
        if p is None:
            if isinstance(dataset, (str, os.PathLike)):
                with open(dataset, "rb") as fh:
                    hdr = fh.read(64)
                p = int.from_bytes(hdr[20:24], "little") if len(hdr) == 64 else 1
            elif isinstance(dataset, (list, tuple)):
                p = int(dataset[0].shape[1])
            else:
                p = int(dataset.shape[1])
        src, keep = self._source(dataset, p, first_row, n_rows, plan)
        starts, counts = plan.partition.arrays()
        res, err = N.ColumnSum(), N.Error()
        st = self._lib.sstat_cuda_column_sum(self._ctx, src, p, column, starts.ctypes.data,
                                             counts.ctypes.data, len(starts), int(plan.precision), flags,
                                             ctypes.byref(res), ctypes.byref(err))
        del keep
        if st == N.ERR_INVALID and "out of range" in err.msg.decode():
            raise IndexError(err.msg.decode())
        if st != N.OK:
            _raise(st, err, in_dataset=True)
        exact = None
        note = None
        if res.exact_ok:
            exact = (res.exact_hi << 64) | res.exact_lo
        else:
            note = f"non-integral value at row {res.note_row}; exact sum unavailable"
        return ColumnSumResult(res.float_sum, exact, bool(res.float_matches_exact), note)

    def comoments(self, dataset, schema: DatasetSchema, plan: ReductionPlan, flags: int = 0, first_row: int = 0,
                  n_rows: Optional[int] = None) -> "CoMoments":
        """run_reduction(accumulate_comoments, merge_comoments) over the plan (suffstats.cpp:107-159)."""
        schema.validate()
        p = schema.column_count()
        src, keep = self._source(dataset, p, first_row, n_rows, plan)
        starts, counts = plan.partition.arrays()
        n, err = ctypes.c_uint64(), N.Error()
        mean, m2 = np.zeros(p), np.zeros(p * (p + 1) // 2)
        dp = ctypes.POINTER(ctypes.c_double)
        st = self._lib.sstat_cuda_comoments(self._ctx, src, p, starts.ctypes.data, counts.ctypes.data,
                                            len(starts), flags, ctypes.byref(n), mean.ctypes.data_as(dp),
                                            m2.ctypes.data_as(dp), ctypes.byref(err))
        del keep
        if st != N.OK:
            _raise(st, err, in_dataset=True)
        return CoMoments(n.value, mean, m2, schema)

    def generate(self, dst, kind: int, seed: int, mu: float, n_int: int, first_row: int, n_rows: int, p: int) -> None:
        """Fill a CUDA tensor with synthetic rows (bit-identical to oracle_generate)."""
        if not _is_torch_cuda(dst):
            raise TypeError("generate needs a CUDA tensor")
        self._check(self._lib.sstat_cuda_generate(self._ctx, ctypes.c_void_p(dst.data_ptr()), kind, seed, mu, n_int,
                                                  first_row, n_rows, p))

    # -- helpers
    @staticmethod
    def _rows_pointer(values, expect: Optional[int]):
        if type(values).__module__.startswith("torch"):
            import torch

            if values.dtype != torch.float64:
                raise TypeError("rows must be float64")
            if not values.is_contiguous():
                raise ValueError("rows must be contiguous row-major")
            if expect is not None and values.numel() != expect:
                raise ValueError("chunk values size does not match row_count * column_count")
            return ctypes.c_void_p(values.data_ptr() or None), values
        arr = np.ascontiguousarray(values, dtype=np.float64)
        if expect is not None and arr.size != expect:
            raise ValueError("chunk values size does not match row_count * column_count")
        return ctypes.c_void_p(arr.ctypes.data if arr.size else None), arr


def _check_width(dataset, p: int) -> None:
    """The rows' width against the schema (check_chunk's width test, suffstats.cpp:33-36):
    2-D inputs must have p columns, flat inputs a multiple of p values."""
    shape = tuple(dataset.shape) if hasattr(dataset, "shape") else np.shape(dataset)
    if len(shape) >= 2:
        bad, cols = shape[-1] != p, shape[-1]
    else:
        numel = int(np.prod(shape)) if shape else 0
        bad, cols = numel % p != 0, numel
    if bad:
        msg = f"range 0 failed: chunk has {cols} columns, schema has {p}"
        raise ReductionError(0, msg, SchemaMismatchError(f"chunk has {cols} columns, schema has {p}"))


def _rows_of(dataset, p: int) -> int:
    numel = dataset.numel() if hasattr(dataset, "numel") else np.asarray(dataset).size
    return int(numel) // p


_default = {}
_default_lock = threading.Lock()


def default_engine(device: Optional[int] = None) -> Engine:
    """Process-wide engine per device (like the reference's free functions)."""
    if device is None:
        try:
            import torch

            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        except Exception:  # pragma: no cover
            device = 0
    with _default_lock:
        if device not in _default:
            _default[device] = Engine(device)
        return _default[device]


def accumulate_chunk(chunk: Chunk, schema: DatasetSchema,
                     precision: PrecisionMode = PrecisionMode.Binary64) -> SuffStats:
    return default_engine().accumulate_chunk(chunk, schema, precision)


def dataset_suffstats(dataset, schema: DatasetSchema, plan: ReductionPlan,
                      timings: Optional[ReductionTimings] = None) -> SuffStats:
    return default_engine().dataset_suffstats(dataset, schema, plan, timings)


def fold_range_partials(partials: np.ndarray, schema: DatasetSchema, plan: ReductionPlan,
                        flags: int = 0) -> SuffStats:
    """The dataset result from all R ranges' partials (R x E, range order) — e.g. checkpointed
    pieces from range_partials — folded on the host in the device's own order (fast mode: the
    32-lane fold; SSTAT_FLAG_REFEXACT / Binary32Diagnostic: the reference's ascending fold), so it
    is bit-identical to dataset_suffstats over the same plan."""
    schema.validate()
    p = schema.column_count()
    R = len(plan.partition.ranges)
    E = p + p * (p + 1) // 2
    parts = np.ascontiguousarray(partials, dtype=np.float64).reshape(-1)
    if parts.size != R * E:
        raise ValueError(f"expected {R} x {E} partials, got {parts.size} values")
    buf = np.concatenate([np.full(4, np.nan), parts])  # one rank: [4-double header | R x E]
    res = np.zeros(E)
    dp = ctypes.POINTER(ctypes.c_double)
    st = N.load().sstat_fold_ranges_host(buf.ctypes.data_as(dp), 4 + R * E, R, 1, p, int(plan.precision), flags,
                                         res.ctypes.data_as(dp))
    if st != N.OK:
        raise ValueError(N.status_string(st))
    out = SuffStats.empty(schema, plan.precision)
    out.n = plan.partition.total_rows()
    out.sums[:] = res[:p]
    out.cross[:] = res[p:]
    return out


def shard_ranges(n_ranges: int, rank: int, world: int):
    """Ranges [first, last) owned by `rank` (contiguous row shards, floor split)."""
    lib = N.load()
    f, l = ctypes.c_uint64(), ctypes.c_uint64()
    st = lib.sstat_shard_ranges(n_ranges, rank, world, ctypes.byref(f), ctypes.byref(l))
    if st != N.OK:
        raise ValueError(N.status_string(st))
    return f.value, l.value
