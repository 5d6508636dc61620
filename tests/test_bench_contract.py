"""bench.py's reference arm on CPU: the JSON line the driver parses (keys, impl, e2e, the
cpu_baseline description) on a small sample, and the non-zero ranks of a torchrun launch."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libsstat_ref.so")


def run_bench(args, env_extra):
    env = dict(os.environ, SSTAT_BENCH_REF_ROWS=str(1_000_000), **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=env, timeout=600, cwd=ROOT)


@pytest.mark.skipif(not os.path.exists(REF_LIB), reason="oracle/_ref not built")
def test_reference_arm_line():
    r = run_bench(["--impl", "reference", "--steps", "2", "--warmup", "1"], {})
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "rows/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["p"] == 16 and d["config"]["rows"] == 1_000_000
    assert d["config"]["same_config"] is False  # shrunk for the test; the driver's run uses the full C2


def test_reference_arm_other_ranks_exit_quietly():
    r = run_bench(["--impl", "reference", "--steps", "1", "--warmup", "1"], {"RANK": "1", "WORLD_SIZE": "2"})
    assert r.returncode == 0 and not [l for l in r.stdout.splitlines() if l.startswith("{")]


def _json_lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_flag_launches_n_ranks(n):
    """bench.py --gpus N outside torchrun re-launches itself with N ranks (torch.distributed.run,
    127.0.0.1); --dry-run runs the launcher and rank plumbing on CPU (gloo): one line, from rank
    0, with n_gpus = N, the max over ranks, and every config's contiguous range shards."""
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--dry-run"],
                       capture_output=True, text=True, env=env, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = _json_lines(r.stdout)
    assert len(lines) == 1, r.stdout
    d = lines[0]
    assert d["dry_run"] and d["n_gpus"] == n and d["max_over_ranks"] == float(n)
    for name, sh in d["shards"].items():
        per = sh["per_rank"]
        assert len(per) == n
        assert per[0][0] == 0 and per[-1][1] == sh["ranges"], name
        assert per[0][2] == 0 and per[-1][3] == sh["rows"], name
        for a, b in zip(per, per[1:]):
            assert a[1] == b[0] and a[3] == b[2], name  # contiguous ranges and rows


def test_gpus_flag_must_match_world_size():
    r = run_bench(["--gpus", "3", "--dry-run"], {"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr
