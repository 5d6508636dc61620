"""Generates tests/golden/golden.json from the UNMODIFIED reference library.

Run in the build container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py

Every expected value comes from the reference itself (oracle/_ref/libsstat_ref.so,
compiled from /root/reference/proj/src by oracle/Makefile).  Inputs are regenerated at
test time by the oracle's generators; their bytes are pinned here by SHA-256 so a
test can tell a generator drift from an accumulation mismatch.  Floats are stored as
float.hex() strings (bit-exact).

Known-answer cases follow the reference's own tests (paths under /root/reference/proj):
  tests/test_suffstats.cpp:45-52   single row -> outer product
  tests/test_suffstats.cpp:54-60   orthogonal rows -> identity
  tests/test_suffstats.cpp:62-74   Table1 seed 21, 10,000 rows, bit-exact vs naive order
  tests/test_suffstats.cpp:100-128 Table1 seed 5, 20,000 rows, chunk 1024, any workers
  tests/test_suffstats.cpp:148-157 inf at row 41, column 1
  tests/test_suffstats.cpp:219-232 binary32 merge rounding
  tests/test_reduce.cpp:36-54      plan_partitions
  tests/test_reduce.cpp:106-168    column_sum KATs
  tests/test_suffstats.cpp:159-172 comoments pairwise algebra
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, Reference  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).reshape(-1)]


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def stats(t):
    n, s, c = t[:3]
    return {"n": int(n), "sums": hx(s), "cross": hx(c)}


def main() -> None:
    o, r = Oracle(), Reference()
    tmp = tempfile.mkdtemp(prefix="sstat_golden_")
    G = {"_source": "reference library built from /root/reference/proj/src (oracle/_ref)", "cases": {}}
    C = G["cases"]

    # -- known answers (test_suffstats.cpp)
    C["single_row"] = {"rows": [[1.0, 2.0]], "p": 2, "start_row": 0, **stats(r.accumulate_chunk(np.array([[1.0, 2.0]]), 2))}
    C["orthogonal"] = {"rows": [[1.0, 0.0], [0.0, 1.0]], "p": 2, "start_row": 0,
                       **stats(r.accumulate_chunk(np.array([[1.0, 0.0], [0.0, 1.0]]), 2))}
    bad = np.array([[1.0, 2.0], [3.0, np.inf]])
    e = r.accumulate_chunk(bad, 2, start_row=40)
    C["nonfinite_chunk"] = {"rows": [[1.0, 2.0], [3.0, "inf"]], "p": 2, "start_row": 40,
                            "error": {"row": e["row"], "col": e["col"], "msg": e["msg"]}}

    t1 = o.table1_chunk(21, 1, 10000)
    C["table1_seed21"] = {"generator": {"table1": True, "seed": 21, "first_index": 1, "n": 10000}, "p": 11,
                          "start_row": 0, "input_sha256": sha(t1), **stats(r.accumulate_chunk(t1, 11))}
    C["table1_seed21_binary32"] = {"generator": {"table1": True, "seed": 21, "first_index": 1, "n": 10000}, "p": 11,
                                   "precision": 1, **stats(r.accumulate_chunk(t1, 11, precision=1))}

    t5 = o.table1_chunk(5, 1, 20000)
    f = os.path.join(tmp, "t5.bin")
    r.write_binary(f, t5, 11)
    ref1 = r.dataset_suffstats(f, 11, 1024, 1)
    ref8 = r.dataset_suffstats(f, 11, 1024, 8)
    assert all(np.array_equal(a, b) for a, b in zip(ref1[1:], ref8[1:]))
    C["table1_seed5_dataset"] = {"generator": {"table1": True, "seed": 5, "first_index": 1, "n": 20000}, "p": 11,
                                 "chunk_rows": 1024, "input_sha256": sha(t5), **stats(ref1)}

    # binary32 merge rounding (test_suffstats.cpp:219-232)
    a32 = r.accumulate_chunk(np.array([[16777216.0]]), 1, precision=1)
    b32 = r.accumulate_chunk(np.array([[1.0]]), 1, precision=1)
    C["binary32_merge"] = {"a": 16777216.0, "b": 1.0, "merged32": hx(r.merge(1, 1, a32, b32)[1])[0],
                           "merged64": hx(r.merge(1, 0, r.accumulate_chunk(np.array([[16777216.0]]), 1),
                                                  r.accumulate_chunk(np.array([[1.0]]), 1))[1])[0]}

    # -- measurement generator cases at oracle-sized n
    gens = {
        "c1_small": dict(kind=1, seed=42, mu=1.0, n_int=0, p=9, n=100000, chunk=1 << 15),
        "c2_small": dict(kind=0, seed=42, mu=1.0, n_int=2, p=16, n=200000, chunk=1 << 16),
        "c2_mu0": dict(kind=0, seed=7, mu=0.0, n_int=2, p=16, n=50000, chunk=4096),
        "ragged_p5": dict(kind=2, seed=3, mu=0.5, n_int=0, p=5, n=9999, chunk=777),
        "p24": dict(kind=0, seed=11, mu=1.0, n_int=3, p=24, n=30001, chunk=5000),
        "p64": dict(kind=0, seed=13, mu=1.0, n_int=4, p=64, n=20000, chunk=4096),
        "wide_p80": dict(kind=2, seed=17, mu=1.0, n_int=0, p=80, n=5000, chunk=2048),
        "wide_p256": dict(kind=2, seed=19, mu=1.0, n_int=0, p=256, n=3000, chunk=1024),
    }
    for name, g in gens.items():
        X = o.generate(g["kind"], g["seed"], g["mu"], g["n_int"], 0, g["n"], g["p"])
        f = os.path.join(tmp, name + ".bin")
        r.write_binary(f, X, g["p"])
        res = r.dataset_suffstats(f, g["p"], g["chunk"], 8)
        case = {"gen": g, "input_sha256": sha(X), **stats(res)}
        ids = [0] if g["kind"] == 1 else []
        an = r.analyze(g["p"], ids, res[0], res[1], res[2])
        iu = np.triu_indices(an[1].shape[0])
        case["analysis"] = {"ids": ids, "mean": hx(an[0]), "cov_upper": hx(an[1][iu]), "corr_upper": hx(an[2][iu])}
        if g["p"] > 64:  # keep the fixture small: wide X^T X is pinned by hash (the oracle recomputes it)
            del case["analysis"]
            case["cross_sha256"] = sha(res[2])
            del case["cross"]
        case["pca_corr_eigenvalues"] = hx(r.run_pca(g["p"], ids, res[0], res[1], res[2], basis=1))
        case["pca_cov_eigenvalues"] = hx(r.run_pca(g["p"], ids, res[0], res[1], res[2], basis=0))
        C[name] = case

    # -- dataset non-finite: lowest failing range, first value in row-major order
    X = o.generate(0, 42, 1.0, 2, 0, 5000, 16)
    X[3000, 5] = np.inf
    X[3000, 9] = np.nan
    X[4500, 1] = np.nan
    f = os.path.join(tmp, "nf.bin")
    r.write_binary(f, X, 16)
    e = r.dataset_suffstats(f, 16, 1024, 4)
    C["dataset_nonfinite"] = {"gen": dict(kind=0, seed=42, mu=1.0, n_int=2, p=16, n=5000, chunk=1024),
                              "poison": [[3000, 5, "inf"], [3000, 9, "nan"], [4500, 1, "nan"]],
                              "error": {"range_index": e["range_index"], "msg": e["msg"]}}

    # -- plan_partitions (test_reduce.cpp:36-54)
    C["plan_partitions"] = {
        str((n, k)): [list(map(int, a)) for a in r.plan_partitions(n, k)] for n, k in [(10, 4), (10, 10), (10000000, 1000000), (5000, 137)]
    }

    # -- column_sum KATs (test_reduce.cpp:106-168), next row #1
    cs = {}
    for name, vals, chunk in [("ids10", "arange:10", 4),
                              ("ids1e5", "arange:100000", 8192),
                              ("flag2p53", [9007199254740992.0, 1.0, 1.0], 3),
                              ("frac", [1.0, 2.5, 3.0], 2),
                              ("ids777", "arange:777", 10)]:
        arr = (np.arange(1, int(vals.split(":")[1]) + 1, dtype=np.float64) if isinstance(vals, str)
               else np.array(vals, dtype=np.float64))
        f = os.path.join(tmp, name + ".bin")
        r.write_binary(f, arr.reshape(-1, 1), 1)
        fs, exact, fm, note = r.column_sum(f, 0, chunk, 3)
        cs[name] = {"values": vals if isinstance(vals, str) else hx(arr), "chunk": chunk, "float_sum": float(fs).hex(),
                    "exact": None if exact is None else str(exact), "float_matches": fm, "note": note}
    C["column_sum"] = cs

    # -- comoments (test_suffstats.cpp:159-172), next row #2
    u = r.accumulate_comoments(np.array([[1.0, 5.0]]), 2)
    v = r.accumulate_comoments(np.array([[3.0, 1.0]]), 2)
    m = r.merge_comoments(2, u, v)
    C["comoments_pair"] = {"n": m[0], "mean": hx(m[1]), "m2": hx(m[2])}

    with open(OUT, "w") as fh:
        json.dump(G, fh, sort_keys=True, separators=(",", ":"))
    print(f"wrote {OUT} ({os.path.getsize(OUT)} bytes, {len(C)} cases)")


if __name__ == "__main__":
    main()
