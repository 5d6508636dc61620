#!/usr/bin/env python
"""Benchmark of the single-pass sufficient-statistics engine (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

`--gpus N` with N > 1 and no torchrun environment re-launches itself under
`torch.distributed.run --nproc-per-node N` (one process per GPU, NCCL); under torchrun,
WORLD_SIZE must equal N.

A step is one dataset_suffstats pass over the rank's HBM-resident shard: the plan's ranges
accumulated (K1), folded per range (K3a), all-gathered over NCCL when N > 1, folded in
ascending range order (K3b) and read back to the host.

Headline workload: config C2 of BASELINE.json — 1e8 rows x 16 FP64 columns per GPU,
HBM-resident, plan_partitions(n, 2^20) (96 ranges per GPU); N > 1 keeps 1e8 rows per GPU (weak
scaling).  Inputs are 12.8 GB per GPU, 100x the 126 MB L2, so no flush is needed between steps.
`value` = global rows / max-over-ranks step time (device events).

Beside it, on the same run (each its own JSON object in the line):
  e2e            the same pass through the public API from pinned host memory (H2D inside every
                 step, result D2H); e2e.file_source = the reference's own call shape,
                 dataset_suffstats(path), on the SSTATBIN bytes in /dev/shm (N = 1);
                 e2e.streamed_c4 = C4's 1.25e9-row shard per GPU (the 1e10-row paper-scale pass
                 over 8 GPUs) streamed through the pinned ring from a pinned host slab (RowReader)
  strong_c3      C3: 1e9 rows x 16 over the N GPUs (strong scaling), with the sha256 of the
                 result bits — identical for every N
  resident_c4    C4: 1.25e9 rows x 16 per GPU, HBM-resident (N = 8: the 1e10-row paper-scale pass),
                 against the aggregate HBM roofline
  c5             C5: 1e8 rows x 256 over the N GPUs (one GPU: a 5e7-row half), the FP64 DMMA
                 SYRK, with its own roofline
  roofline       the accumulate kernel of the headline pass: algorithmic bytes (rows x 8p, read
                 once) per launch / its CUDA-event duration, against MEASURED_PEAKS.json
  cpu_baseline   the reference's own dataset_suffstats (oracle/_ref, built from /root/reference)
                 on the SAME C2 bytes (N = 1), all host threads, plus the parity of our result
                 against it (parity_c2_vs_reference)
  next_rows      column_sum and co-moments on the resident C2 shard (N = 1)
  c1             C1, the reference's CPU-runnable case (1e6 x (8 + ID), one range, N = 1): the
                 call time through the API and the accumulate kernel's, L2 flushed (a 256 MB read)
                 before every call

--impl reference runs only the CPU reference arm (rank 0) on the C2 bytes and prints its line.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rows/sec (and HBM GB/s, % roofline) of sufficient-stats pass, 1/2/4/8 B200 vs CPU"
CHUNK_ROWS = 1 << 20
SEED, MU = 42, 1.0
C2_ROWS, C2_P = 100_000_000, 16
C3_ROWS = 1_000_000_000
C4_ROWS_PER_GPU = 1_250_000_000
C5_ROWS, C5_P = 100_000_000, 256
DMMA_PEAK_TFLOPS = 37.03  # measured: profiles/r01_fp64_probe.log (mma.sync m8n8k4 f64, 148 SMs)
TOL = 1e-12


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_of(kernel_key):
    """DRAM bytes per launch of a kernel from the committed ncu --set full capture of its
    workload (profiles/traffic.json, written by tools/summarize_profiles.py): a static copy."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f)
        if kernel_key in tr:
            return tr[kernel_key]["dram_read_bytes"] + tr[kernel_key]["dram_write_bytes"], tr[kernel_key].get("source")
    except Exception:
        pass
    return None, None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (host time, fields)
        self.window = None
        self._proc = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                           "--format=csv,noheader,nounits", "-lms", "20"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            for line in self._proc.stdout:
                self.rows.append((time.perf_counter(), [x.strip() for x in line.strip().split(",")]))
        except Exception:
            pass

    def start(self):
        self._t.start()
        time.sleep(0.3)  # nvidia-smi needs a moment before its first line

    def mark(self, t0: float, t1: float):
        self.window = (t0, t1)

    def stop(self):
        if self._proc is not None:
            self._proc.terminate()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows or self.window is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        t0, t1 = self.window
        inside = [r for t, r in self.rows if t0 <= t <= t1]
        note = "samples inside the timed region"
        if len(inside) < 3:  # short timed region: widen to the adjacent warm-up/drain samples
            inside = [r for t, r in self.rows if t0 - 0.25 <= t <= t1 + 0.25]
            note = "timed region +-0.25 s (region shorter than the 20 ms sampling period x 3)"
        sm = [float(r[0]) for r in inside if r and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in inside if len(r) > 1 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in inside for i in range(4) if len(r) > 3 + i and r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(inside), "note": note}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def host_info() -> dict:
    """CPU model, thread count and RAM of this host (stated beside the CPU timing)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        ram = 0
    return {"cpu": model, "nproc": os.cpu_count() or 1, "ram_gb": round(ram / 1e9, 1)}


def shm_dir() -> str:
    return "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()


def sstatbin_header(n: int, p: int) -> bytes:
    hdr = bytearray(64)
    hdr[0:8] = b"SSTATBIN"
    hdr[8:12] = (1).to_bytes(4, "little")
    hdr[12:20] = int(n).to_bytes(8, "little")
    hdr[20:24] = int(p).to_bytes(4, "little")
    return bytes(hdr)


def sha_bits(ss) -> str:
    import numpy as np

    h = hashlib.sha256()
    h.update(np.int64(ss.n).tobytes())
    h.update(np.ascontiguousarray(ss.sums).tobytes())
    h.update(np.ascontiguousarray(ss.cross).tobytes())
    return h.hexdigest()


def cs_errors(got_sums, got_cross, n, ref_sums, ref_cross, p):
    """Cauchy-Schwarz-normalised errors: max |dS_jk| / sqrt(S_jj S_kk) and
    max |ds_j| / sqrt(n S_jj)."""
    import numpy as np

    iu = np.triu_indices(p)
    diag = np.array([ref_cross[j * p - j * (j - 1) // 2] for j in range(p)])
    scale = np.sqrt(np.abs(diag[iu[0]] * diag[iu[1]]))
    scale[scale == 0] = 1.0
    s_scale = np.sqrt(np.abs(n * diag))
    s_scale[s_scale == 0] = 1.0
    return (float(np.max(np.abs(got_cross - ref_cross) / scale)),
            float(np.max(np.abs(got_sums - ref_sums) / s_scale)))


# ------------------------------------------------------------------ the CPU reference
def write_c2_file_oracle(path: str, rows: int, p: int, workers: int) -> None:
    """The C2 bytes (SplitMix64 RowRng generator, 2 integer + 14 Gaussian columns) written by
    the oracle's C generator in parallel slabs — bit-identical to the GPU generator."""
    import numpy as np
    from concurrent.futures import ThreadPoolExecutor

    from oracle.oracle import Oracle

    orc = Oracle()
    slab = 1_000_000
    with open(path, "wb") as f:
        f.write(sstatbin_header(rows, p))

        def gen(s):
            return orc.generate(0, SEED, MU, 2, s, min(slab, rows - s), p)

        with ThreadPoolExecutor(workers) as ex:
            for arr in ex.map(gen, range(0, rows, slab)):
                f.write(np.ascontiguousarray(arr).tobytes())


def reference_passes(path: str, p: int, passes: int, workers: int):
    """The reference's own dataset_suffstats (oracle/_ref, the unmodified library) over the
    SSTATBIN file, plan_partitions(n, 2^20), `workers` threads (reduce.cpp:90-98).  Returns the
    per-pass wall times, the last pass's result and read / work split."""
    from oracle.oracle import Reference

    ref = Reference()
    times, res = [], None
    for _ in range(passes):
        t0 = time.perf_counter()
        res = ref.dataset_suffstats(path, p, CHUNK_ROWS, workers, 0, timings=True)
        times.append(time.perf_counter() - t0)
        if isinstance(res, dict):
            raise RuntimeError(res)
    return times, res


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    # the full C2 bytes; SSTAT_BENCH_REF_ROWS shrinks them for the CPU test suite only
    rows = int(os.environ.get("SSTAT_BENCH_REF_ROWS", C2_ROWS))
    path = os.path.join(shm_dir(), f"sstat_ref_c2_{os.getpid()}.bin")
    try:
        write_c2_file_oracle(path, rows, C2_P, workers)
        times, res = reference_passes(path, C2_P, args.warmup + args.steps, workers)
    finally:
        try:
            os.remove(path)
        except OSError:
            pass
    timed = times[args.warmup:]
    v = rows / statistics.median(timed)
    info = host_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(timed),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64 RowRng generator, bit-identical to the GPU inputs)",
        "config": {"workload": f"C2: the reference's dataset_suffstats over the {rows:.0e} x 16 SSTATBIN file "
                               f"({rows * 128 / 1e9:.1f} GB in /dev/shm, page cache), plan_partitions(n, 2^20) = "
                               f"{-(-rows // CHUNK_ROWS)} ranges, {workers} worker threads", "rows": rows, "p": C2_P,
                   "ranges": -(-rows // CHUNK_ROWS), "same_config": world == 1 and rows == C2_ROWS,
                   "note": None if world == 1 else f"CPU arm times the 1e8-row C2 pass (the per-GPU shard) "
                                                    f"for the N={world} line"},
        "gb_per_s": v * 8 * C2_P / 1e9,
        "cpu_baseline": {"value": v, "unit": "rows/s", "cores": workers, "kind": "reference", **info,
                         "sample": f"the C2 bytes ({rows} rows x {C2_P}), one dataset_suffstats pass per "
                                   f"step, median of {len(timed)}; last pass read {res[3]:.2f} s / work "
                                   f"{res[4]:.2f} s summed over workers"},
        "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def relaunch_under_torchrun(args) -> int:
    """--gpus N outside torchrun: one process per GPU through torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, RowReader, plan_partitions, shard_ranges

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        # the communicators' own log lines (transport, rings / NVLS), on stderr: stdout carries the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def shard_of(n_global):
        pl = ReductionPlan(plan_partitions(n_global, CHUNK_ROWS))
        R = len(pl.partition.ranges)
        f, l = shard_ranges(R, rank, world)
        r0 = pl.partition.ranges[f].start_row
        r1 = pl.partition.ranges[l - 1].start_row + pl.partition.ranges[l - 1].row_count
        return pl, r0, r1 - r0

    eng = Engine(local)
    eng.collect_timings = True  # K1's CUDA-event time for the roofline; the kernel name
    if world > 1:
        obj = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng.init_distributed(rank, world, obj[0])
    stream = torch.cuda.current_stream()
    eng.set_stream(stream.cuda_stream)

    def device_timed(fn, k, warm=2):
        for _ in range(warm):
            fn()
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        out = None
        for _ in range(k):
            out = fn()
        b.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b) / k * 1e-3), out

    # ---------------- headline: C2 per GPU (weak scaling) ----------------
    p = C2_P
    n_global = C2_ROWS * world
    plan, r0, local_rows = shard_of(n_global)
    R = len(plan.partition.ranges)
    schema = DatasetSchema.generic(p, False)
    D = torch.empty((local_rows, p), dtype=torch.float64, device="cuda")
    eng.generate(D, 0, SEED, MU, 2, r0, local_rows, p)
    torch.cuda.synchronize()

    def step():
        return eng.dataset_suffstats(D, schema, plan, first_row=r0, n_rows=local_rows)

    for _ in range(max(args.warmup, 3)):
        step()
    kern, launches = [], 0
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_start = time.perf_counter()
    e0.record(stream)
    for _ in range(args.steps):
        res = step()
        kern.append(eng.last_timings.kernel_seconds)
        launches += eng.last_timings.kernel_launches
    e1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(t_start, time.perf_counter())
    barrier()
    clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    kern_s = max_over_ranks(sum(kern) / len(kern))
    k1_name = eng.last_timings.kernel.decode()
    value = n_global / (ms * 1e-3)
    c2_result = res

    # ---------------- SURVEY §8(f) rows on the resident shard (one GPU) ----------------
    next_rows = None
    if not args.no_next and world == 1:
        k_next = max(3, min(args.steps, 10))
        t_cs, _ = device_timed(lambda: eng.column_sum(D, 0, plan, p=p, first_row=r0, n_rows=local_rows), k_next)
        t_cm, _ = device_timed(lambda: eng.comoments(D, schema, plan, first_row=r0, n_rows=local_rows), k_next)
        next_rows = {
            "column_sum": {"value": n_global / t_cs, "unit": "rows/s", "ms_per_step": t_cs * 1e3, "column": 0,
                           "what": "column_sum (reduce.cpp:32-88): FP64 sum + exact 128-bit integer sum of one column",
                           "column_gb_per_s": local_rows * 8 / t_cs / 1e9,
                           # bytes the memory system must move per row for one 8-B column: the
                           # whole row while it fits one 128-B line (ncu at C2: DRAM read = all 8p
                           # bytes), else at least one 32-B sector
                           "moved_gb_per_s": local_rows * (8 * p if 8 * p <= 128 else 32) / t_cs / 1e9},
            "comoments": {"value": n_global / t_cm, "unit": "rows/s", "ms_per_step": t_cm * 1e3,
                          "what": "run_reduction(accumulate_comoments, merge_comoments) (suffstats.cpp:107-159)",
                          "gb_per_s": local_rows * p * 8 / t_cm / 1e9},
        }

    # ---------------- C1: 1e6 x (8 + ID), one range (the reference's CPU-runnable case) ----------------
    c1_line = None
    if not args.no_c1 and world == 1:
        n1, p1 = 1_000_000, 9
        D1 = torch.empty((n1, p1), dtype=torch.float64, device="cuda")
        eng.generate(D1, 1, SEED, MU, 0, 0, n1, p1)
        plan1 = ReductionPlan(plan_partitions(n1, CHUNK_ROWS))
        sc1 = DatasetSchema.generic(p1, True)
        # L2 flush by a 256 MB read (> the 126 MB L2) before every call: clean lines, so the call
        # neither finds its rows in L2 nor pays for another buffer's write-backs
        flush = torch.ones(32 << 20, dtype=torch.float64, device="cuda")
        k1s, calls, calls_timed = [], [], []
        for timed in (False, True):
            eng.collect_timings = timed
            for it in range(205):
                flush.sum()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                eng.dataset_suffstats(D1, sc1, plan1)
                b.record(stream)
                torch.cuda.synchronize()
                if it >= 5:
                    (calls_timed if timed else calls).append(a.elapsed_time(b) * 1e3)
                    if timed:
                        k1s.append(eng.last_timings.kernel_seconds * 1e6)
        eng.collect_timings = True
        med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
        k1_us = med(k1s)
        hbm_peak, _ = peaks()
        c1_line = {"rows": n1, "p": p1, "ranges": 1, "value": n1 / (med(calls) * 1e-6), "unit": "rows/s",
                   "call_us": med(calls), "call_us_with_timings": med(calls_timed), "k1_us": k1_us,
                   "k1_gb_per_s": n1 * p1 * 8 / (k1_us * 1e-6) / 1e9,
                   "k1_frac": n1 * p1 * 8 / (k1_us * 1e-6) / 1e9 / hbm_peak,
                   "kernel": eng.last_timings.kernel.decode(), "calls": len(calls),
                   "l2": "flushed before every call (a 256 MB read)",
                   "k1_note": "k1_us by the two graph event nodes around K1 (a few us of node time at this size; "
                              "ncu's cold capture: 20.7 us, profiles/r02_k1_c1_full.md)",
                   "what": "dataset_suffstats(CUDA tensor) of 1e6 rows x (8 + ID): K1 on one wave of tiles, K3a, "
                           "read-back, one replayed graph; call_us = device time from before the call to after "
                           "its return (medians over 200 calls)"}
        del D1, flush
        torch.cuda.empty_cache()

    # ---------------- e2e: the public API from pinned host memory ----------------
    e2e, cpu, parity, H = None, None, None, None
    shard_bytes = local_rows * p * 8
    info = host_info()
    fits = info["ram_gb"] > 0 and world * shard_bytes <= 0.45 * info["ram_gb"] * 1e9
    if not args.no_e2e and not fits:
        e2e = {"unavailable": f"{world} x {shard_bytes / 1e9:.1f} GB pinned shards exceed 45 % of the "
                              f"{info['ram_gb']:.0f} GB host RAM"}
    if not args.no_e2e and fits:
        H = torch.empty((local_rows, p), dtype=torch.float64, pin_memory=True)
        H.copy_(D)
        del D
        torch.cuda.empty_cache()
        eng.set_stream(0)
        for _ in range(2):
            got = eng.dataset_suffstats(H, schema, plan, first_row=r0, n_rows=local_rows)
        assert got.bit_equal(c2_result), "host-streamed result differs from the HBM-resident one"
        k_e2e = max(2, min(args.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            got = eng.dataset_suffstats(H, schema, plan, first_row=r0, n_rows=local_rows)
        dt = max_over_ranks((time.perf_counter() - t0) / k_e2e)
        barrier()
        E = p + p * (p + 1) // 2
        e2e = {"value": n_global / dt, "unit": "rows/s", "h2d_bytes_per_step": shard_bytes,
               "d2h_bytes_per_step": (E + 4 * world) * 8, "steps": k_e2e, "ms_per_step": dt * 1e3,
               "h2d_gb_per_s_per_gpu": shard_bytes / dt / 1e9,
               "what": "dataset_suffstats(pinned host tensor): 4-slot pinned ring, H2D on a copy stream || "
                       "K1 on the compute stream, K3a/K3b, result D2H"}

        # the SSTATBIN bytes of the shard in /dev/shm: the reference's call shape through our
        # engine, and (one GPU) the reference itself on the same bytes
        if world == 1:
            path = os.path.join(shm_dir(), f"sstat_c2_{os.getpid()}.bin")
            try:
                with open(path, "wb") as f:
                    f.write(sstatbin_header(local_rows, p))
                    H.numpy().tofile(f)
                got = eng.dataset_suffstats(path, schema, plan)
                assert got.bit_equal(c2_result), "file-source result differs from the HBM-resident one"
                t0 = time.perf_counter()
                for _ in range(k_e2e):
                    eng.dataset_suffstats(path, schema, plan)
                dt = (time.perf_counter() - t0) / k_e2e
                e2e["file_source"] = {
                    "value": local_rows / dt, "unit": "rows/s", "file_bytes": 64 + shard_bytes, "steps": k_e2e,
                    "ms_per_step": dt * 1e3, "gb_per_s": shard_bytes / dt / 1e9,
                    "host_threads": min(16, os.cpu_count() or 1),
                    "what": "dataset_suffstats(SSTATBIN path in /dev/shm): parallel pread feeder -> pinned "
                            "staging -> H2D -> K1 -> K3 -> result D2H"}
                if not args.no_cpu:
                    workers = os.cpu_count() or 1
                    times, ref = reference_passes(path, p, 4, workers)
                    v = local_rows / statistics.median(times[1:])
                    cpu = {"value": v, "unit": "rows/s", "cores": workers, "kind": "reference", **info,
                           "sample": f"the same C2 bytes ({local_rows} rows x {p}, SSTATBIN in /dev/shm), the "
                                     f"reference's dataset_suffstats with {workers} threads, median of 3 passes "
                                     f"after 1 warm-up; last pass read {ref[3]:.2f} s / work {ref[4]:.2f} s "
                                     f"summed over workers", "same_config": True}
                    parity = c2_parity(c2_result, ref, p)
            finally:
                try:
                    os.remove(path)
                except OSError:
                    pass

        # C4: the rank's 1.25e9-row shard streamed from a pinned slab (the C2 shard, reused at
        # advancing row offsets) through the RowReader callback
        if not args.no_c4:
            e2e["streamed_c4"] = streamed_c4(eng, H, schema, world, rank, max_over_ranks, barrier)
        eng.set_stream(stream.cuda_stream)
    if H is not None:
        del H
    else:
        del D
    torch.cuda.empty_cache()

    # ---------------- C3: 1e9 rows over the N GPUs (strong scaling) ----------------
    strong = None
    if not args.no_c3:
        pl3, q0, nq = shard_of(C3_ROWS)
        D3 = torch.empty((nq, p), dtype=torch.float64, device="cuda")
        eng.generate(D3, 0, SEED, MU, 2, q0, nq, p)
        torch.cuda.synchronize()
        k3 = max(3, min(args.steps, 10))
        t3, r3 = device_timed(lambda: eng.dataset_suffstats(D3, schema, pl3, first_row=q0, n_rows=nq), k3)
        strong = {"value": C3_ROWS / t3, "unit": "rows/s", "ms_per_step": t3 * 1e3, "steps": k3,
                  "global_rows": C3_ROWS, "rows_per_gpu": nq, "ranges": len(pl3.partition.ranges),
                  "gb_per_s": C3_ROWS * p * 8 / t3 / 1e9,
                  "hbm_frac": C3_ROWS * p * 8 / t3 / 1e9 / (world * peaks()[0]),
                  "result_sha256": sha_bits(r3),
                  "what": "C3: 1e9 x 16 row-sharded across the GPUs, rank-ordered all-gather of per-range partials, "
                          "ascending range fold; the result bits (sha256) are the same for every N"}
        del D3
        torch.cuda.empty_cache()

    # ---------------- C4 resident: 1.25e9 rows x 16 per GPU (N = 8: the 1e10-row paper-scale
    # pass, the north star's >= 85 % of aggregate HBM target) ----------------
    c4 = None
    if not args.no_c4:
        n4 = C4_ROWS_PER_GPU * world
        pl4, q0, nq = shard_of(n4)
        D4 = torch.empty((nq, p), dtype=torch.float64, device="cuda")
        eng.generate(D4, 0, SEED, MU, 2, q0, nq, p)
        torch.cuda.synchronize()
        k4 = max(3, min(args.steps, 5))
        kern4 = []

        def step4():
            r = eng.dataset_suffstats(D4, schema, pl4, first_row=q0, n_rows=nq)
            kern4.append(eng.last_timings.kernel_seconds)
            return r

        t4, r4 = device_timed(step4, k4)
        k4_s = max_over_ranks(sum(kern4[-k4:]) / k4)
        peak, _ = peaks()
        c4 = {"value": n4 / t4, "unit": "rows/s", "ms_per_step": t4 * 1e3, "steps": k4, "global_rows": n4,
              "rows_per_gpu": nq, "ranges": len(pl4.partition.ranges), "gb_per_s": n4 * p * 8 / t4 / 1e9,
              "hbm_frac_aggregate": n4 * p * 8 / t4 / 1e9 / (world * peak),
              "kernel_frac": nq * p * 8 / k4_s / 1e9 / peak, "result_sha256": sha_bits(r4),
              "what": "C4 HBM-resident: 1.25e9 x 16 per GPU (160 GB), the whole pass (K1, folds, exchange, "
                      "read-back) against N x the measured copy peak; at N = 8 this is the 1e10-row paper-scale "
                      "pass of the north star"}
        del D4
        torch.cuda.empty_cache()

    # ---------------- C5: 1e8 x 256 over the N GPUs (one GPU: a 5e7-row half) ----------------
    c5 = None
    if not args.no_c5:
        rows5 = C5_ROWS if world > 1 else C5_ROWS // 2
        pl5, q0, nq = (shard_of(rows5))
        D5 = torch.empty((nq, C5_P), dtype=torch.float64, device="cuda")
        eng.generate(D5, 2, SEED, MU, 0, q0, nq, C5_P)
        torch.cuda.synchronize()
        sc5 = DatasetSchema.generic(C5_P, False)
        k5 = max(3, min(args.steps, 5))
        kern5 = []

        def step5():
            r = eng.dataset_suffstats(D5, sc5, pl5, first_row=q0, n_rows=nq)
            kern5.append(eng.last_timings.kernel_seconds)
            return r

        t5, r5 = device_timed(step5, k5)
        k5_s = max_over_ranks(sum(kern5[-k5:]) / k5)
        flops = nq * C5_P * (C5_P + 2)
        traffic, tsrc = traffic_of("k_widep")
        c5 = {"value": rows5 / t5, "unit": "rows/s", "ms_per_step": t5 * 1e3, "steps": k5, "global_rows": rows5,
              "rows_per_gpu": nq, "p": C5_P, "ranges": len(pl5.partition.ranges),
              "tflops": rows5 * C5_P * (C5_P + 2) / t5 / 1e12, "result_sha256": sha_bits(r5),
              "workload": "C5: 1e8 x 256 FP64 Gaussian" + (" over the GPUs" if world > 1 else
                                                           ": a 5e7-row half (204.8 GB does not fit one GPU)"),
              "roofline": {"bound": "tensor", "achieved": flops / k5_s / 1e12, "peak": DMMA_PEAK_TFLOPS,
                           "unit": "TFLOP/s", "frac": flops / k5_s / 1e12 / DMMA_PEAK_TFLOPS,
                           "traffic": traffic, "traffic_source": tsrc,
                           "kernel": eng.last_timings.kernel.decode(), "per_launch_flops": flops,
                           "per_launch_ms": k5_s * 1e3,
                           "peak_source": "measured FP64 DMMA peak (profiles/r01_fp64_probe.log; MEASURED_PEAKS.json "
                                          "has no FP64 entry)"}}
        del D5
        torch.cuda.empty_cache()

    if rank == 0:
        peak, peak_src = peaks()
        traffic, tsrc = traffic_of("k_smallp")
        achieved = shard_bytes / kern_s / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": tsrc, "kernel": k1_name, "per_launch_bytes": shard_bytes,
                "per_launch_ms": kern_s * 1e3, "peak_source": peak_src}
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (bit-portable SplitMix64 RowRng generator, same bytes as the CPU oracle)",
            "config": {"workload": "C2: 1e8 rows x 16 FP64 cols per GPU (2 integer rand_between(1,100) + 14 "
                                   "Gaussian, mu=1), HBM-resident", "rows_per_gpu": local_rows,
                       "global_rows": n_global, "p": p, "chunk_rows": CHUNK_ROWS, "ranges": R,
                       "l2": f"no flush: {shard_bytes / 1e9:.1f} GB/GPU inputs are >>126 MB L2",
                       "parallelism": f"{world} GPU row shards" + (", NCCL all-gather of per-range partials"
                                                                   if world > 1 else "")},
            "gb_per_s": value * 8 * p / 1e9,
            "roofline": roof,
            "cpu_baseline": cpu,
            "parity_c2_vs_reference": parity,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "result_sha256": sha_bits(c2_result),
            "strong_c3": strong,
            "resident_c4": c4,
            "c5": c5,
            "next_rows": next_rows,
            "c1": c1_line,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def c2_parity(got, ref, p):
    """Our C2 result against the reference's own dataset_suffstats on the same bytes (SURVEY
    §8(d) tolerances): integer block bit-exact, FP64 sums / X^T X Cauchy-Schwarz-normalised
    <= 1e-12, and the reference's analyze / run_pca on both results (cov / corr / eigenvalues)."""
    import numpy as np

    from oracle.oracle import Reference

    rn, rs, rS = ref[0], ref[1], ref[2]
    ints = [0, 1]  # rand_between(1, 100) columns
    idx = [j * p - j * (j - 1) // 2 + (k - j) for j in ints for k in ints if k >= j]
    int_exact = bool(np.array_equal(got.sums[ints].view(np.uint64), rs[ints].view(np.uint64)) and
                     np.array_equal(got.cross[idx].view(np.uint64), rS[idx].view(np.uint64)))
    cs, se = cs_errors(got.sums, got.cross, got.n, rs, rS, p)
    ref_lib = Reference()
    m_a, cov_a, corr_a = ref_lib.analyze(p, [], got.n, got.sums, got.cross)
    m_b, cov_b, corr_b = ref_lib.analyze(p, [], rn, rs, rS)
    dcov = float(np.max(np.abs(cov_a - cov_b) / np.sqrt(np.outer(np.diag(cov_b), np.diag(cov_b)))))
    dcorr = float(np.max(np.abs(corr_a - corr_b)))
    ev_a = ref_lib.run_pca(p, [], got.n, got.sums, got.cross)
    ev_b = ref_lib.run_pca(p, [], rn, rs, rS)
    dev = float(np.max(np.abs(ev_a - ev_b) / np.abs(ev_b)))
    ok = got.n == rn and int_exact and cs <= TOL and se <= TOL and dcov <= TOL and dcorr <= TOL and dev <= 1e-10
    return {"ok": bool(ok), "n_equal": got.n == rn, "integer_block_bit_exact": int_exact, "cross_cs_err": cs,
            "sums_err": se, "cov_cs_err": dcov, "corr_abs_err": dcorr, "eig_rel_err": dev,
            "bars": "integer bit-exact; S, sums, cov 1e-12 (Cauchy-Schwarz normalised); corr 1e-12 abs; "
                    "eigenvalues 1e-10 rel",
            "what": "GPU fast path vs the reference's dataset_suffstats (oracle/_ref) on the same 12.8 GB"}


def streamed_c4(eng, H, schema, world, rank, max_over_ranks, barrier):
    """C4 per GPU: the rank's 1.25e9-row shard of the 1e10-row dataset, streamed through the
    4-slot pinned ring.  1.28 TB does not fit host RAM, so the rows come from a RowReader that
    serves the pinned C2 slab at advancing row offsets (row r reads slab row r mod S; a chunk
    that wraps is copied into the pinned scratch slot).  Every byte still crosses PCIe once.
    Check: the integer columns' entries are exact and known — 12.5 slabs' worth."""
    import ctypes

    import numpy as np
    import torch

    from paper_2604_23826_b200 import ReductionPlan, RowReader, plan_partitions, shard_ranges

    rows, p = H.shape
    rb = p * 8
    # the period: whole staging slots (256 MiB, 2^21 rows at p = 16), so a slot never wraps
    slot_rows = (256 << 20) // rb
    S = max(slot_rows, rows // slot_rows * slot_rows)
    n_global = C4_ROWS_PER_GPU * world
    plan = ReductionPlan(plan_partitions(n_global, CHUNK_ROWS))
    R = len(plan.partition.ranges)
    f, l = shard_ranges(R, rank, world)
    r0 = plan.partition.ranges[f].start_row
    nloc = plan.partition.ranges[l - 1].start_row + plan.partition.ranges[l - 1].row_count - r0
    base = H.data_ptr()

    def read(row, k, scratch):
        off = (row - r0) % S
        if off + k <= S:
            return base + off * rb
        first = S - off
        ctypes.memmove(scratch, base + off * rb, first * rb)
        ctypes.memmove(scratch + first * rb, base, (k - first) * rb)
        return scratch

    reader = RowReader(read, n_rows=nloc, first_row=r0)  # the rank's rows
    res = eng.dataset_suffstats(reader, schema, plan)  # warm-up (and the check below)
    # expected integer entries: the slab's exact integer sums, times whole periods + the partial one
    full, rem = divmod(nloc, S)
    X = H[:S, :2].numpy().astype(np.int64)
    Xr = X[:rem]
    want_s = full * X.sum(axis=0) + Xr.sum(axis=0)
    want_c = [full * int((X[:, j] * X[:, k]).sum()) + int((Xr[:, j] * Xr[:, k]).sum()) for j, k in ((0, 0), (0, 1), (1, 1))]
    exact = world > 1 or (res.n == nloc and [float(v) for v in want_s] == [float(v) for v in res.sums[:2]] and
                          [float(v) for v in want_c] == [res.cross[0], res.cross[1], res.cross[p]])
    k = 2
    barrier()
    t0 = time.perf_counter()
    for _ in range(k):
        eng.dataset_suffstats(reader, schema, plan)
    dt = max_over_ranks((time.perf_counter() - t0) / k)
    barrier()
    del torch
    return {"value": n_global / dt, "unit": "rows/s", "rows_per_gpu": nloc, "global_rows": n_global, "steps": k,
            "ms_per_step": dt * 1e3, "h2d_bytes_per_step_per_gpu": nloc * rb,
            "gb_per_s_per_gpu": nloc * rb / dt / 1e9, "gb_per_s_aggregate": n_global * rb / dt / 1e9,
            "integer_entries_exact": bool(exact) if world == 1 else "checked on one GPU",
            "what": "C4 shard (1.25e9 x 16 per GPU) through dataset_suffstats(RowReader): a pinned slab of "
                    f"{S} rows served at advancing offsets (period = whole 256 MiB slots) -> 4-slot pinned ring "
                    "-> H2D -> K1 -> K3 -> D2H"}


def run_dry(args):
    """--dry-run: the launcher and the multi-rank plumbing on CPU (gloo): the rank layout of
    every config's plan (contiguous range shards, sstat_shard_ranges) and the max-over-ranks
    reduction, with no device work.  Rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist

    from paper_2604_23826_b200 import ReductionPlan, plan_partitions, shard_ranges

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    shards = {}
    for name, n in (("c2", C2_ROWS * world), ("c3", C3_ROWS), ("c4", C4_ROWS_PER_GPU * world),
                    ("c5", C5_ROWS if world > 1 else C5_ROWS // 2)):
        pl = ReductionPlan(plan_partitions(n, CHUNK_ROWS))
        R = len(pl.partition.ranges)
        f, l = shard_ranges(R, rank, world)
        mine = (f, l, pl.partition.ranges[f].start_row,
                pl.partition.ranges[l - 1].start_row + pl.partition.ranges[l - 1].row_count)
        allr = [None] * world
        if world > 1:
            dist.all_gather_object(allr, mine)
        else:
            allr = [mine]
        shards[name] = {"rows": n, "ranges": R, "per_rank": allr}
    t = torch.tensor([float(rank + 1)])
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "max_over_ranks": float(t.item()), "shards": shards}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the column_sum / co-moment timings")
    ap.add_argument("--no-c3", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 call-time leg")
    ap.add_argument("--dry-run", action="store_true", help="launcher + rank layout only, CPU (gloo)")
    args = ap.parse_args()
    world_env = os.environ.get("WORLD_SIZE")
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if world_env is None and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    if world_env is not None and int(world_env) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
