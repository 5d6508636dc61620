"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and an ncu
--set full report into profiles/<tag>_*.  Usage:
    python tools/summarize_profiles.py <tag> gpurun_out/launches.csv gpurun_out/k1_full.ncu-rep
"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "gpc__cycles_elapsed.avg.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__ops_path_tensor_src_fp64.sum",
    "lts__t_bytes.sum", "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum",
]


def launches(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr = rows[0]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        agg[r[i_name].replace("(anonymous namespace)::", "").split("(")[0]].append(float(r[i_val].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | total ms | avg us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e3:.1f} | {100 * sum(v) / tot:.1f}% |")
    return "\n".join(out)


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"### `{name}`\n\n| metric | value | unit |\n|---|---:|---|")
        for i, h in enumerate(hdr):
            if h in KEYS:
                out.append(f"| {h} | {vals[i]} | {units[i]} |")
    return "\n".join(out)


def traffic(rep):
    """dram read/write bytes of the captured launch (for bench.py's roofline.traffic)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def get(name):
        i = hdr.index(name)
        return float(vals[i].replace(",", "")) * scale[units[i]]

    return {"dram_read_bytes": get("dram__bytes_read.sum"), "dram_write_bytes": get("dram__bytes_write.sum")}


if __name__ == "__main__":
    tag, lc, rep = sys.argv[1:4]
    with open(f"profiles/{tag}_launches.md", "w") as f:
        f.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none, cold & serialised)\n\n")
        f.write("Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py "
                "--steps 2 --warmup 3 --no-e2e --no-cpu --no-next`\n\n")
        f.write(launches(lc) + "\n")
    with open(f"profiles/{tag}_k1_full.md", "w") as f:
        f.write(f"# {tag}: ncu --set full of the accumulate kernel (one launch, C2 1e8 x 16)\n\n")
        f.write(full(rep) + "\n")
    print(open(f"profiles/{tag}_launches.md").read())
