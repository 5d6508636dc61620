"""Summarise ncu output into profiles/ (tracked):
  * a launch list (ncu --metrics gpu__time_duration.sum[,dram__bytes_*] --csv): per-kernel launches,
    average duration, share of the profiled time, DRAM bytes per launch;
  * --set full reports: the key metrics of each captured launch, and (--traffic key) the captured
    launch's DRAM bytes into profiles/traffic.json for bench.py's roofline.traffic.
Usage:
    python tools/summarize_profiles.py launches <out.md> <launches.csv> "<command>"
    python tools/summarize_profiles.py full <out.md> <report.ncu-rep> "<title>" [--traffic key "workload"]
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.avg.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "launch__cluster_dim_x", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__ops_path_tensor_src_fp64.sum",
    "lts__t_bytes.sum", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launch_table(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    i_id, i_name, i_m, i_u, i_v = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Unit",
                                                           "Metric Value"))
    per = defaultdict(dict)  # (id, kernel) -> metric -> value
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        v = float(r[i_v].replace(",", "")) * SCALE.get(r[i_u], 1)
        per[(r[i_id], r[i_name].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0].replace("void ", ""))][r[i_m]] = v
    agg = defaultdict(list)
    for (_, k), m in per.items():
        agg[k].append(m)
    tot = sum(m.get("gpu__time_duration.sum", 0) for v in agg.values() for m in v)
    out = ["| kernel | launches | avg us | share | DRAM read / launch | DRAM write / launch |",
           "|---|---:|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1])):
        t = sum(m.get("gpu__time_duration.sum", 0) for m in v)
        rd = sum(m.get("dram__bytes_read.sum", 0) for m in v) / len(v)
        wr = sum(m.get("dram__bytes_write.sum", 0) for m in v) / len(v)
        out.append(f"| `{k}` | {len(v)} | {t / len(v) / 1e3:.1f} | {100 * t / tot:.1f}% | {rd / 1e9:.4f} GB | "
                   f"{wr / 1e9:.4f} GB |")
    return "\n".join(out)


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    return rows[0], rows[1], rows[2:]


def full_table(rep):
    hdr, units, launches = raw(rep)
    out = []
    for vals in launches:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"### `{name}`\n\n| metric | value | unit |\n|---|---:|---|")
        for i, h in enumerate(hdr):
            if h in KEYS:
                out.append(f"| {h} | {vals[i]} | {units[i]} |")
    return "\n".join(out)


def update_traffic(rep, key, workload, source):
    hdr, units, launches = raw(rep)
    vals = launches[0]

    def get(name):
        i = hdr.index(name)
        return float(vals[i].replace(",", "")) * SCALE[units[i]]

    path = os.path.join(ROOT, "profiles", "traffic.json")
    tr = json.load(open(path)) if os.path.exists(path) else {}
    tr[key] = {"dram_read_bytes": get("dram__bytes_read.sum"), "dram_write_bytes": get("dram__bytes_write.sum"),
               "duration_ms": get("gpu__time_duration.sum") / 1e6 if units[hdr.index("gpu__time_duration.sum")] == "ns"
               else None, "source": source, "workload": workload}
    json.dump(tr, open(path, "w"), indent=1)


if __name__ == "__main__":
    mode, out = sys.argv[1], sys.argv[2]
    if mode == "launches":
        csv_path, cmd = sys.argv[3], sys.argv[4]
        with open(out, "w") as f:
            f.write(f"# ncu launch list (--clock-control none: cold, serialised launches)\n\nCommand: `{cmd}`\n\n")
            f.write(launch_table(csv_path) + "\n")
    else:
        rep, title = sys.argv[3], sys.argv[4]
        with open(out, "w") as f:
            f.write(f"# {title}\n\n" + full_table(rep) + "\n")
        if "--traffic" in sys.argv:
            i = sys.argv.index("--traffic")
            update_traffic(rep, sys.argv[i + 1], sys.argv[i + 2], os.path.relpath(out, ROOT))
    print(open(out).read())
