"""ctypes access to the test oracles.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs (cpu_baseline and
--impl reference) may import this module — as the checker or the CPU baseline,
never as the product path.

  Oracle      liboracle.so: C restatement of the reference path (sstat_oracle.c)
  Reference   _ref/libsstat_ref.so: the unmodified reference library + ref_shim.cpp
              (built from /root/reference by oracle/Makefile; travels to the GPU box)
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, Structure, byref, c_char, c_char_p, c_double, c_int, c_int64, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsstat_ref.so")
REF_SRC = "/root/reference/proj"

dp = POINTER(c_double)
u64p = POINTER(c_uint64)
u32p = POINTER(c_uint32)

NONFINITE = 1


def build(ref: bool = True) -> None:
    """Compile liboracle.so, and the reference library when its sources are present."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _d(a: np.ndarray):
    return a.ctypes.data_as(dp)


class Oracle:
    """The C restatement (sstat_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = ctypes.CDLL(path)
        L.oracle_accumulate_chunk.argtypes = [dp, c_uint64, c_uint32, c_uint64, c_uint32, u64p, dp, dp, u64p, u32p]
        L.oracle_merge.argtypes = [c_uint32, c_uint32, u64p, dp, dp, c_uint64, dp, dp]
        L.oracle_plan_partitions.restype = c_uint64
        L.oracle_plan_partitions.argtypes = [c_uint64, c_uint64, c_void_p, c_void_p]
        L.oracle_run_reduction.argtypes = [dp, c_uint32, c_uint32, c_void_p, c_void_p, c_uint64, c_uint32, u64p, dp, dp,
                                           u64p, u64p, u32p]
        L.oracle_generated_reduction.argtypes = [c_uint32, c_uint64, c_double, c_uint32, c_uint32, c_void_p, c_void_p,
                                                 c_uint64, c_uint32, u64p, dp, dp]
        L.oracle_generate.argtypes = [c_uint32, c_uint64, c_double, c_uint32, c_uint64, c_uint64, c_uint32, dp]
        L.oracle_table1_chunk.argtypes = [c_uint64, c_uint64, c_uint64, dp]
        L.oracle_iid_row.argtypes = [c_uint64, c_uint64, c_uint32, c_double, c_double, dp]
        L.oracle_rowrng_u64.restype = c_uint64
        L.oracle_rowrng_u64.argtypes = [c_uint64, c_uint64, c_uint64]
        L.oracle_column_sum.argtypes = [dp, c_uint32, c_uint32, c_uint32, c_void_p, c_void_p, c_uint64, dp,
                                        POINTER(c_int), POINTER(c_int64), u64p, u64p]
        L.oracle_accumulate_comoments.argtypes = [dp, c_uint64, c_uint32, c_uint64, u64p, dp, dp, u64p, u32p]
        L.oracle_merge_comoments.argtypes = [c_uint32, u64p, dp, dp, c_uint64, dp, dp]
        self.L = L

    # --- accumulate_chunk / merge / fold
    def accumulate_chunk(self, values: np.ndarray, p: int, start_row: int = 0, precision: int = 0):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        rows = v.size // p
        n = c_uint64()
        sums = np.zeros(p)
        cross = np.zeros(p * (p + 1) // 2)
        er, ec = c_uint64(), c_uint32()
        st = self.L.oracle_accumulate_chunk(_d(v), rows, p, start_row, precision, byref(n), _d(sums), _d(cross),
                                            byref(er), byref(ec))
        if st == NONFINITE:
            return ("nonfinite", er.value, ec.value)
        assert st == 0, st
        return n.value, sums, cross

    def plan_partitions(self, n_rows: int, chunk_rows: int):
        R = self.L.oracle_plan_partitions(n_rows, chunk_rows, None, None)
        s = np.zeros(R, dtype=np.uint64)
        c = np.zeros(R, dtype=np.uint64)
        self.L.oracle_plan_partitions(n_rows, chunk_rows, s.ctypes.data, c.ctypes.data)
        return s, c

    def run_reduction(self, values: np.ndarray, p: int, starts, counts, workers: int = 1, precision: int = 0):
        """run_reduction over in-memory rows; ('nonfinite', range, row, col) on failure."""
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        s = np.ascontiguousarray(starts, dtype=np.uint64)
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        n = c_uint64()
        sums = np.zeros(p)
        cross = np.zeros(p * (p + 1) // 2)
        erange, erow, ecol = c_uint64(), c_uint64(), c_uint32()
        st = self.L.oracle_run_reduction(_d(v), p, precision, s.ctypes.data, c.ctypes.data, len(s), workers, byref(n),
                                         _d(sums), _d(cross), byref(erange), byref(erow), byref(ecol))
        if st == NONFINITE:
            return ("nonfinite", erange.value, erow.value, ecol.value)
        assert st == 0, st
        return n.value, sums, cross

    def generated_reduction(self, kind, seed, mu, n_int, p, starts, counts, workers):
        s = np.ascontiguousarray(starts, dtype=np.uint64)
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        n = c_uint64()
        sums = np.zeros(p)
        cross = np.zeros(p * (p + 1) // 2)
        self.L.oracle_generated_reduction(kind, seed, mu, n_int, p, s.ctypes.data, c.ctypes.data, len(s), workers,
                                          byref(n), _d(sums), _d(cross))
        return n.value, sums, cross

    def merge(self, p, precision, a, b):
        n = c_uint64(a[0])
        sa, ca = a[1].copy(), a[2].copy()
        self.L.oracle_merge(p, precision, byref(n), _d(sa), _d(ca), b[0], _d(np.ascontiguousarray(b[1])),
                            _d(np.ascontiguousarray(b[2])))
        return n.value, sa, ca

    # --- generators
    def generate(self, kind: int, seed: int, mu: float, n_int: int, first_row: int, n_rows: int, p: int) -> np.ndarray:
        out = np.empty((n_rows, p))
        self.L.oracle_generate(kind, seed, mu, n_int, first_row, n_rows, p, _d(out))
        return out

    def table1_chunk(self, seed: int, first_index: int, n: int) -> np.ndarray:
        out = np.empty((n, 11))
        self.L.oracle_table1_chunk(seed, first_index, n, _d(out))
        return out

    def iid_row(self, seed, index, p, lo, hi):
        out = np.empty(p + 1)
        self.L.oracle_iid_row(seed, index, p, lo, hi, _d(out))
        return out

    def rowrng_u64(self, seed, row_index, position):
        return self.L.oracle_rowrng_u64(seed, row_index, position)

    # --- next rows
    def column_sum(self, values, p, column, starts, counts, precision=0):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        s = np.ascontiguousarray(starts, dtype=np.uint64)
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        fs, ok, hi, lo, nrow = c_double(), c_int(), c_int64(), c_uint64(), c_uint64()
        self.L.oracle_column_sum(_d(v), p, column, precision, s.ctypes.data, c.ctypes.data, len(s), byref(fs),
                                 byref(ok), byref(hi), byref(lo), byref(nrow))
        exact = (hi.value << 64) | lo.value if ok.value else None
        return fs.value, exact, (nrow.value if not ok.value else None)

    def accumulate_comoments(self, values, p, start_row=0):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        n = c_uint64()
        mean = np.zeros(p)
        m2 = np.zeros(p * (p + 1) // 2)
        er, ec = c_uint64(), c_uint32()
        st = self.L.oracle_accumulate_comoments(_d(v), v.size // p, p, start_row, byref(n), _d(mean), _d(m2), byref(er),
                                                byref(ec))
        assert st == 0
        return n.value, mean, m2

    def merge_comoments(self, p, a, b):
        n = c_uint64(a[0])
        ma, m2a = a[1].copy(), a[2].copy()
        self.L.oracle_merge_comoments(p, byref(n), _d(ma), _d(m2a), b[0], _d(np.ascontiguousarray(b[1])),
                                      _d(np.ascontiguousarray(b[2])))
        return n.value, ma, m2a


class RefError(Structure):
    _fields_ = [("row", c_uint64), ("col", c_uint32), ("range_index", c_uint64), ("msg", c_char * 256)]


class Reference:
    """The unmodified reference library (oracle/_ref/libsstat_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing and /root/reference is not available to build it")
        L = ctypes.CDLL(path)
        E = POINTER(RefError)
        L.ref_accumulate_chunk.argtypes = [dp, c_uint64, c_uint32, c_uint64, c_uint32, u64p, dp, dp, E]
        L.ref_merge.argtypes = [c_uint32, c_uint32, u64p, dp, dp, c_uint64, dp, dp]
        L.ref_write_binary.argtypes = [c_char_p, dp, c_uint64, c_uint32, c_int, E]
        L.ref_dataset_suffstats.argtypes = [c_char_p, c_uint32, c_uint64, c_uint32, c_uint32, u64p, dp, dp, dp, dp, E]
        L.ref_dataset_suffstats_ranges.argtypes = [c_char_p, c_uint32, c_void_p, c_void_p, c_uint64, c_uint32, u64p, dp,
                                                   dp, E]
        L.ref_plan_partitions.restype = c_uint64
        L.ref_plan_partitions.argtypes = [c_uint64, c_uint64, c_void_p, c_void_p, E]
        L.ref_generate_row.argtypes = [c_int, c_uint64, c_double, c_double, c_uint64, c_uint64, dp]
        L.ref_column_sum.argtypes = [c_char_p, c_uint32, c_uint64, c_uint32, c_uint32, dp, POINTER(c_int),
                                     POINTER(c_int64), u64p, POINTER(c_int), c_char_p, E]
        L.ref_accumulate_comoments.argtypes = [dp, c_uint64, c_uint32, c_uint64, u64p, dp, dp, E]
        L.ref_merge_comoments.argtypes = [c_uint32, u64p, dp, dp, c_uint64, dp, dp]
        L.ref_analyze.argtypes = [c_uint32, c_uint32, u32p, c_uint64, dp, dp, c_int, u32p, dp, dp, dp, POINTER(c_int), E]
        L.ref_run_pca.argtypes = [c_uint32, c_uint32, u32p, c_uint64, dp, dp, c_int, u32p, dp, E]
        L.ref_save_suffstats.argtypes = [c_char_p, c_uint32, c_uint32, u32p, c_uint32, c_uint64, dp, dp, E]
        self.L = L

    @staticmethod
    def _err(st, e):
        return {"status": st, "row": e.row, "col": e.col, "range_index": e.range_index, "msg": e.msg.decode()}

    def accumulate_chunk(self, values, p, start_row=0, precision=0):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        n = c_uint64()
        sums, cross = np.zeros(p), np.zeros(p * (p + 1) // 2)
        e = RefError()
        st = self.L.ref_accumulate_chunk(_d(v), v.size // p, p, start_row, precision, byref(n), _d(sums), _d(cross),
                                         byref(e))
        if st:
            return self._err(st, e)
        return n.value, sums, cross

    def merge(self, p, precision, a, b):
        n = c_uint64(a[0])
        sa, ca = a[1].copy(), a[2].copy()
        st = self.L.ref_merge(p, precision, byref(n), _d(sa), _d(ca), b[0], _d(np.ascontiguousarray(b[1])),
                              _d(np.ascontiguousarray(b[2])))
        assert st == 0
        return n.value, sa, ca

    def write_binary(self, path, values, p, with_checksum=True):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        e = RefError()
        st = self.L.ref_write_binary(os.fsencode(path), _d(v), v.size // p, p, int(with_checksum), byref(e))
        if st:
            raise RuntimeError(self._err(st, e))

    def dataset_suffstats(self, path, p, chunk_rows=1 << 20, workers=1, precision=0, timings=False):
        n = c_uint64()
        sums, cross = np.zeros(p), np.zeros(p * (p + 1) // 2)
        rs, ws = c_double(), c_double()
        e = RefError()
        st = self.L.ref_dataset_suffstats(os.fsencode(path), p, chunk_rows, workers, precision, byref(n), _d(sums),
                                          _d(cross), byref(rs), byref(ws), byref(e))
        if st:
            return self._err(st, e)
        if timings:
            return n.value, sums, cross, rs.value, ws.value
        return n.value, sums, cross

    def dataset_suffstats_ranges(self, path, p, starts, counts, workers=1):
        s = np.ascontiguousarray(starts, dtype=np.uint64)
        c = np.ascontiguousarray(counts, dtype=np.uint64)
        n = c_uint64()
        sums, cross = np.zeros(p), np.zeros(p * (p + 1) // 2)
        e = RefError()
        st = self.L.ref_dataset_suffstats_ranges(os.fsencode(path), p, s.ctypes.data, c.ctypes.data, len(s), workers,
                                                 byref(n), _d(sums), _d(cross), byref(e))
        if st:
            return self._err(st, e)
        return n.value, sums, cross

    def plan_partitions(self, n_rows, chunk_rows):
        e = RefError()
        R = self.L.ref_plan_partitions(n_rows, chunk_rows, None, None, byref(e))
        s = np.zeros(R, dtype=np.uint64)
        c = np.zeros(R, dtype=np.uint64)
        self.L.ref_plan_partitions(n_rows, chunk_rows, s.ctypes.data, c.ctypes.data, byref(e))
        return s, c

    def generate_row(self, kind, seed, index, iid_columns=10, lo=0.0, hi=1.0):
        out = np.empty(11 if kind == 0 else iid_columns + 1)
        self.L.ref_generate_row(kind, iid_columns, lo, hi, seed, index, _d(out))
        return out

    def column_sum(self, path, column, chunk_rows, workers=1, precision=0):
        fs, ok, hi, lo, fm = c_double(), c_int(), c_int64(), c_uint64(), c_int()
        note = ctypes.create_string_buffer(256)
        e = RefError()
        st = self.L.ref_column_sum(os.fsencode(path), column, chunk_rows, workers, precision, byref(fs), byref(ok),
                                   byref(hi), byref(lo), byref(fm), note, byref(e))
        if st:
            return self._err(st, e)
        exact = (hi.value << 64) | lo.value if ok.value else None
        return fs.value, exact, bool(fm.value), note.value.decode()

    def accumulate_comoments(self, values, p, start_row=0):
        v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        n = c_uint64()
        mean, m2 = np.zeros(p), np.zeros(p * (p + 1) // 2)
        e = RefError()
        st = self.L.ref_accumulate_comoments(_d(v), v.size // p, p, start_row, byref(n), _d(mean), _d(m2), byref(e))
        assert st == 0
        return n.value, mean, m2

    def merge_comoments(self, p, a, b):
        n = c_uint64(a[0])
        ma, m2a = a[1].copy(), a[2].copy()
        self.L.ref_merge_comoments(p, byref(n), _d(ma), _d(m2a), b[0], _d(np.ascontiguousarray(b[1])),
                                   _d(np.ascontiguousarray(b[2])))
        return n.value, ma, m2a

    def analyze(self, p, ids, n, sums, cross, ddof=1):
        idarr = np.ascontiguousarray(ids, dtype=np.uint32)
        q = c_uint32()
        mean, cov, corr = np.zeros(p), np.zeros(p * p), np.zeros(p * p)
        ok = c_int()
        e = RefError()
        st = self.L.ref_analyze(p, len(idarr), idarr.ctypes.data_as(u32p), n, _d(np.ascontiguousarray(sums)),
                                _d(np.ascontiguousarray(cross)), ddof, byref(q), _d(mean), _d(cov), _d(corr), byref(ok),
                                byref(e))
        if st:
            return self._err(st, e)
        m = q.value
        return mean[:m], cov[: m * m].reshape(m, m), (corr[: m * m].reshape(m, m) if ok.value else None)

    def run_pca(self, p, ids, n, sums, cross, basis=1):
        idarr = np.ascontiguousarray(ids, dtype=np.uint32)
        q = c_uint32()
        ev = np.zeros(p)
        e = RefError()
        st = self.L.ref_run_pca(p, len(idarr), idarr.ctypes.data_as(u32p), n, _d(np.ascontiguousarray(sums)),
                                _d(np.ascontiguousarray(cross)), basis, byref(q), _d(ev), byref(e))
        if st:
            return self._err(st, e)
        return ev[: q.value]
