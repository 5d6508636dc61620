"""One driver for the A/B experiments of the tuning logs in profiles/ (replaces the one-shot
shell scripts of round 1): for every variant (a label and SSTAT_* environment overrides) run
the width sweep (tools/p_sweep.py) or the step timer (tools/step_time.py), optionally followed
by a pytest selection under the same environment.

    python tools/ab_sweep.py --widths 136,152,160 \\
        --variant default --variant "wg0r3:SSTAT_WIDEP_WG=0,SSTAT_WIDEP_R=3" [--tests "-k wide_p"]
    python tools/ab_sweep.py --step --variant "tr512:SSTAT_K1_TILE_ROWS=512" --variant default
"""
import argparse
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def parse_variant(v):
    label, _, assigns = v.partition(":")
    env = {}
    for a in filter(None, assigns.split(",")):
        k, _, val = a.partition("=")
        env[k.strip()] = val.strip()
    return label, env


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", action="append", default=[], help="label[:VAR=value,VAR=value]")
    ap.add_argument("--widths", default="", help="p values for tools/p_sweep.py")
    ap.add_argument("--bytes", default="8e9", help="input bytes per width (p_sweep)")
    ap.add_argument("--step", action="store_true", help="time C1 / C2 steps (tools/step_time.py) instead")
    ap.add_argument("--tests", default="", help="pytest arguments run under every variant (-m gpu implied)")
    ap.add_argument("--timeout", type=int, default=600)
    args = ap.parse_args()
    for v in args.variant or ["default"]:
        label, env_over = parse_variant(v)
        env = dict(os.environ, **env_over)
        print(f"== {label} {env_over}", flush=True)
        if args.step:
            cmd = [sys.executable, os.path.join(HERE, "step_time.py"), "200"]
        else:
            env["SWEEP_P"] = args.widths
            cmd = [sys.executable, os.path.join(HERE, "p_sweep.py"), args.bytes]
        r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=args.timeout)
        print(r.stdout.rstrip(), flush=True)
        if r.returncode:
            print(f"   rc={r.returncode}: {r.stderr[-500:]}", flush=True)
        if args.tests:
            t = subprocess.run([sys.executable, "-m", "pytest", "tests", "-q", "-x", "-m", "gpu"] + args.tests.split(),
                               env=env, cwd=ROOT, capture_output=True, text=True, timeout=args.timeout * 3)
            print("   pytest: " + (t.stdout.strip().splitlines() or ["?"])[-1], flush=True)


if __name__ == "__main__":
    main()
