#!/usr/bin/env python
"""Benchmark of the single-pass sufficient-statistics engine (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c2|c1|c3]

A step is one dataset_suffstats pass over the rank's HBM-resident shard: the plan's
ranges accumulated (K1), folded per range (K3a), all-gathered over NCCL when N > 1,
folded in ascending range order (K3b) and read back to the host.

Workload (N=1): config C2 of BASELINE.json — 1e8 rows x 16 FP64 columns, HBM-resident,
plan_partitions(n, 2^20) (96 ranges).  N > 1 keeps 1e8 rows per GPU (weak scaling;
global n = N x 1e8, rows sharded contiguously by range).  Inputs are 12.8 GB per GPU,
100x the 126 MB L2, so no flush is needed between steps.

`value` = global rows / max-over-ranks step time (device events).  `e2e` = the same
pass through the public API from pinned host memory (H2D inside every step, result
D2H); `e2e.file_source` = the reference's own call shape, dataset_suffstats(path), on an
SSTATBIN copy in /dev/shm read by the parallel host feeder.  `roofline` = the accumulate kernel K1: algorithmic bytes (rows x 8p, read once)
per launch / its average CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
`cpu_baseline` = the reference's own dataset_suffstats (oracle/_ref, built from
/root/reference) on a bounded sample, on this host's cores.

--impl reference runs only that CPU reference arm (rank 0) and prints its line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "rows/sec (and HBM GB/s, % roofline) of sufficient-stats pass, 1/2/4/8 B200 vs CPU"
CONFIGS = {
    # name: (rows per GPU, p, generator kind, integer columns, description)
    "c2": (100_000_000, 16, 0, 2, "C2: 1e8 rows x 16 FP64 cols per GPU (2 integer rand_between(1,100) + 14 "
                                   "Gaussian, mu=1), HBM-resident"),
    "c1": (1_000_000, 9, 1, 0, "C1: 1e6 rows x (8 FP64 Gaussian + 1 ID) per GPU, HBM-resident"),
    "c3": (125_000_000, 16, 0, 2, "C3 shard: 1.25e8 rows x 16 per GPU (1e9 over 8 GPUs), HBM-resident"),
    "c4": (1_250_000_000, 16, 0, 2, "C4 shard: 1.25e9 rows x 16 per GPU (160 GB; the 1e10-row paper-scale pass "
                                    "over 8 GPUs), HBM-resident"),
    "c5": (50_000_000, 256, 2, 0, "C5 shard: 5e7 rows x 256 FP64 Gaussian cols per GPU (the 1e8 x 256 = 204.8 GB "
                                  "config over 2 GPUs), HBM-resident, FP64 DMMA SYRK"),
}
DMMA_PEAK_TFLOPS = 37.03  # measured: profiles/r01_fp64_probe.log (mma.sync m8n8k4 f64, 148 SMs)
CHUNK_ROWS = 1 << 20
SEED, MU = 42, 1.0
# reference CPU arm sample: 2.56 GB SSTATBIN in /dev/shm (2e7 rows at p=16); the override is for tests
CPU_SAMPLE_BYTES = int(os.environ.get("SSTAT_BENCH_SAMPLE_BYTES", 2_560_000_000))


def cpu_sample_rows(p: int) -> int:
    return CPU_SAMPLE_BYTES // (8 * p)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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


def cpu_model() -> str:
    """The host CPU model string (report it beside the CPU timing)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_rows_per_s(steps: int, warmup: int, config: str = "c2"):
    """The reference's own dataset_suffstats (oracle/_ref) on a 2.56 GB SSTATBIN sample of the
    config's workload (same generator, same p, chunk 2^20), all host threads.  Returns
    (per-step rows/s, threads, (read s, work s), sample rows)."""
    _, p, kind, n_int, _ = CONFIGS[config]
    sample_rows = cpu_sample_rows(p)
    import numpy as np

    from oracle.oracle import Oracle, Reference

    ref, orc = Reference(), Oracle()
    workers = os.cpu_count() or 1
    d = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
    path = os.path.join(d, f"sstat_bench_{os.getpid()}.bin")
    try:
        # write the sample in slabs (oracle generator, bit-identical to the GPU generator)
        import ctypes

        with open(path, "wb") as f:
            hdr = bytearray(64)
            hdr[0:8] = b"SSTATBIN"
            hdr[8:12] = (1).to_bytes(4, "little")
            hdr[12:20] = sample_rows.to_bytes(8, "little")
            hdr[20:24] = p.to_bytes(4, "little")
            f.write(hdr)
            slab = 1_000_000
            from concurrent.futures import ThreadPoolExecutor

            def gen(s):
                return orc.generate(kind, SEED, MU, n_int, s, min(slab, sample_rows - s), p)

            with ThreadPoolExecutor(workers) as ex:
                for arr in ex.map(gen, range(0, sample_rows, slab)):
                    f.write(np.ascontiguousarray(arr).tobytes())
        rates = []
        split = None
        for i in range(warmup + steps):
            t0 = time.perf_counter()
            res = ref.dataset_suffstats(path, p, CHUNK_ROWS, workers, 0, timings=True)
            dt = time.perf_counter() - t0
            if isinstance(res, dict):
                raise RuntimeError(res)
            if i >= warmup:
                rates.append(sample_rows / dt)
                split = (res[3], res[4])
        return rates, workers, split, sample_rows
    finally:
        try:
            os.remove(path)
        except OSError:
            pass


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    rates, cores, split, sample = cpu_reference_rows_per_s(args.steps, args.warmup, args.config)
    v = statistics.median(rates)
    rows, p, *_ = CONFIGS[args.config]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "rows/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sample / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64 RowRng generator, bit-identical to the GPU inputs)",
        "config": {"workload": f"reference CPU dataset_suffstats on a {sample:.2e}-row sample of "
                               f"{args.config.upper()} (p={p}, chunk_rows 2^20, SSTATBIN in page cache)",
                   "p": p, "sample_rows": sample},
        "gb_per_s": v * 8 * p / 1e9,
        "cpu_baseline": {"value": v, "unit": "rows/s", "cores": cores, "kind": "reference", "cpu": cpu_model(),
                         "sample": f"{sample} rows x {p} of the {args.config.upper()} generator, one "
                                   f"dataset_suffstats pass per step, {cores} worker threads; "
                                   f"last step read {split[0]:.2f} s / work {split[1]:.2f} s (summed over workers)"},
        "e2e": {"value": v, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def e2e_file_source(eng, H, schema, plan, ref_res, steps):
    """The reference's own call shape, dataset_suffstats(path, schema, plan), on an SSTATBIN
    copy of the shard in /dev/shm (page cache, as the reference arm reads it): parallel
    feeder reads into pinned staging + H2D + kernels + result D2H, timed on the host."""
    import numpy as np

    n, p = H.shape
    d = "/dev/shm" if os.path.isdir("/dev/shm") else tempfile.gettempdir()
    path = os.path.join(d, f"sstat_e2e_{os.getpid()}.bin")
    try:
        hdr = bytearray(64)
        hdr[0:8] = b"SSTATBIN"
        hdr[8:12] = (1).to_bytes(4, "little")
        hdr[12:20] = int(n).to_bytes(8, "little")
        hdr[20:24] = int(p).to_bytes(4, "little")
        with open(path, "wb") as f:
            f.write(hdr)
            H.numpy().tofile(f)
        got = eng.dataset_suffstats(path, schema, plan)
        assert got.bit_equal(ref_res), "file-source result differs from the HBM-resident one"
        t0 = time.perf_counter()
        for _ in range(steps):
            eng.dataset_suffstats(path, schema, plan)
        dt = (time.perf_counter() - t0) / steps
        return {"value": n / dt, "unit": "rows/s", "file_bytes": 64 + n * p * 8, "steps": steps,
                "ms_per_step": dt * 1e3, "gb_per_s": n * p * 8 / dt / 1e9,
                "host_threads": min(16, os.cpu_count() or 1),
                "what": "dataset_suffstats(SSTATBIN path in /dev/shm): parallel pread feeder -> pinned "
                        "staging -> H2D -> K1 -> K3 -> result D2H"}
    except OSError as e:
        return {"unavailable": str(e)}
    finally:
        try:
            os.remove(path)
        except OSError:
            pass


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2604_23826_b200 import DatasetSchema, Engine, ReductionPlan, plan_partitions, shard_ranges

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rows_per_gpu, p, kind, n_int, desc = CONFIGS[args.config]
    n_global = rows_per_gpu * world
    plan = ReductionPlan(plan_partitions(n_global, CHUNK_ROWS))
    R = len(plan.partition.ranges)
    f, l = shard_ranges(R, rank, world)
    r0 = plan.partition.ranges[f].start_row
    r1 = plan.partition.ranges[l - 1].start_row + plan.partition.ranges[l - 1].row_count
    local_rows = r1 - r0
    schema = DatasetSchema.generic(p, kind == 1)

    eng = Engine(local)
    if world > 1:
        obj = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng.init_distributed(rank, world, obj[0])
    stream = torch.cuda.current_stream()
    eng.set_stream(stream.cuda_stream)

    D = torch.empty((local_rows, p), dtype=torch.float64, device="cuda")
    eng.generate(D, kind, SEED, MU, n_int, r0, local_rows, p)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

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
    value = n_global / (ms * 1e-3)

    # ---- SURVEY §8(f) rows on the same resident shard: column_sum (exact identifier sum)
    # and co-moments, device-timed like the main pass ----
    def timed(fn, k):
        for _ in range(2):
            fn()
        barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(k):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return max_over_ranks(a.elapsed_time(b) / k * 1e-3)

    next_rows = None
    if not args.no_next and world == 1:  # the §8(f) rows are measured on one GPU
        k_next = max(3, min(args.steps, 10))
        t_cs = timed(lambda: eng.column_sum(D, 0, plan, p=p, first_row=r0, n_rows=local_rows), k_next)
        t_cm = timed(lambda: eng.comoments(D, schema, plan, first_row=r0, n_rows=local_rows), k_next)
        next_rows = {
            "column_sum": {"value": n_global / t_cs, "unit": "rows/s", "ms_per_step": t_cs * 1e3, "column": 0,
                           "what": "column_sum (reduce.cpp:32-88): FP64 sum + exact 128-bit integer sum of one column",
                           "column_gb_per_s": local_rows * 8 / t_cs / 1e9,
                           # bytes the memory system must move per row for one 8-B column: the
                           # whole row while it fits one 128-B line (ncu at C2: 4 L2 sectors per
                           # row, DRAM read = all 8p bytes), else at least one 32-B sector
                           "moved_gb_per_s": local_rows * (8 * p if 8 * p <= 128 else 32) / t_cs / 1e9,
                           "note": "row-major rows: one 8-B column costs the whole row up to 128-B rows "
                                   "(C2: the bound is the row bytes at HBM bandwidth) and at least a 32-B "
                                   "sector per row beyond"},
            "comoments": {"value": n_global / t_cm, "unit": "rows/s", "ms_per_step": t_cm * 1e3,
                          "what": "run_reduction(accumulate_comoments, merge_comoments) (suffstats.cpp:107-159)",
                          "gb_per_s": local_rows * p * 8 / t_cm / 1e9},
        }

    # ---- e2e: public API from pinned host memory (H2D + result D2H every step) ----
    e2e = None
    # the e2e leg needs every rank's shard in pinned host memory at once: only when all of them
    # fit in half the node's RAM (no pageable intermediate copy)
    shard_bytes = local_rows * p * 8
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        ram = 0
    fits = ram > 0 and world * shard_bytes <= 0.5 * ram
    if not args.no_e2e and not fits:
        e2e = {"unavailable": f"{world} x {shard_bytes / 1e9:.1f} GB pinned shards exceed half of the "
                              f"{ram / 1e9:.0f} GB host RAM"}
    if not args.no_e2e and fits and p <= 64 and shard_bytes <= 32e9:
        H = torch.empty((local_rows, p), dtype=torch.float64, pin_memory=True)
        H.copy_(D)
        del D
        torch.cuda.empty_cache()
        eng.set_stream(0)
        ref_res = res
        for _ in range(2):
            got = eng.dataset_suffstats(H, schema, plan, first_row=r0, n_rows=local_rows)
        assert got.bit_equal(ref_res), "host-streamed result differs from the HBM-resident one"
        k_e2e = max(2, min(args.steps, 5))
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            got = eng.dataset_suffstats(H, schema, plan, first_row=r0, n_rows=local_rows)
        dt = max_over_ranks((time.perf_counter() - t0) / k_e2e)
        barrier()
        E = p + p * (p + 1) // 2
        e2e = {"value": n_global / dt, "unit": "rows/s", "h2d_bytes_per_step": local_rows * p * 8,
               "d2h_bytes_per_step": (E + 4 * world) * 8, "steps": k_e2e, "ms_per_step": dt * 1e3,
               "h2d_gb_per_s_per_gpu": local_rows * p * 8 / dt / 1e9}
        if world == 1:
            e2e["file_source"] = e2e_file_source(eng, H, schema, plan, ref_res, k_e2e)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rates, cores, split, sample = cpu_reference_rows_per_s(steps=3, warmup=1, config=args.config)
        cpu = {"value": statistics.median(rates), "unit": "rows/s", "cores": cores, "kind": "reference", "cpu": cpu_model(),
               "sample": f"reference dataset_suffstats (oracle/_ref) over {sample} rows x {p} of the same "
                         f"generator, chunk_rows 2^20, {cores} worker threads, median of 3 passes"}

    if rank == 0:
        peak, peak_src = peaks()
        # dram bytes per launch of the dominant kernel from the committed ncu --set full capture
        # of this workload (profiles/traffic.json; written by tools/summarize_profiles.py)
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tr = json.load(f)
            key = {"c2": "k_smallp", "c5": "k_widep"}.get(args.config) if world == 1 else None
            if key in tr:
                traffic = tr[key]["dram_read_bytes"] + tr[key]["dram_write_bytes"]
        except Exception:
            traffic = None
        bytes_per_launch = local_rows * p * 8
        achieved = bytes_per_launch / kern_s / 1e9
        if p > 64:  # compute-bound: FP64 tensor-pipe roofline, p(p+2) flops per row
            flops = local_rows * p * (p + 2)
            roof = {"bound": "tensor", "achieved": flops / kern_s / 1e12, "peak": DMMA_PEAK_TFLOPS,
                    "unit": "TFLOP/s", "frac": flops / kern_s / 1e12 / DMMA_PEAK_TFLOPS, "traffic": traffic,
                    "kernel": "k_widep (K2)", "per_launch_flops": flops, "per_launch_ms": kern_s * 1e3,
                    "peak_source": "measured FP64 DMMA peak (profiles/r01_fp64_probe.log; MEASURED_PEAKS.json "
                                   "has no FP64 entry)", "hbm_gb_per_s": achieved}
        else:
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "kernel": f"k_smallp<{(p + 7) // 8},{str(p % 16 == 0).lower()}> (K1)",
                    "per_launch_bytes": bytes_per_launch, "per_launch_ms": kern_s * 1e3, "peak_source": peak_src}
        line = {
            "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (bit-portable SplitMix64 RowRng generator, same bytes as the CPU oracle)",
            "config": {"workload": desc, "rows_per_gpu": local_rows, "global_rows": n_global, "p": p,
                       "chunk_rows": CHUNK_ROWS, "ranges": R,
                       "l2": f"no flush: {local_rows * p * 8 / 1e9:.1f} GB/GPU inputs are >>126 MB L2",
                       "parallelism": f"{world} GPU row shards" + (", NCCL all-gather of per-range partials"
                                                                   if world > 1 else "")},
            "gb_per_s": value * 8 * p / 1e9,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
            "next_rows": next_rows,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-next", action="store_true", help="skip the column_sum / co-moment timings")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
