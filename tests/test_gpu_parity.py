"""GPU parity: the CUDA path (through the C ABI) against the reference's own results.

Bars (BASELINE.json north_star):
  * counts: exact; integer-valued columns: bit-exact (all partial sums < 2^53);
  * FP64 sums / X^T X: Cauchy-Schwarz-normalised error <= 1e-12
        |dS_jk| <= 1e-12 sqrt(S_jj S_kk),  |ds_j| <= 1e-12 sqrt(n S_jj);
  * covariance (CS-normalised) and correlation (absolute) <= 1e-12, eigenvalues 1e-10 relative;
  * SSTAT_FLAG_REFEXACT (and Binary32Diagnostic): bit-identical to the reference for any data.
"""
from __future__ import annotations

import hashlib
import os

import numpy as np
import pytest

from conftest import bits, cs_err, sums_err, truth_suffstats, unhex

pytestmark = pytest.mark.gpu

TOL = 1e-12


def torch_mod():
    import torch

    return torch


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def schema(p, ids=()):
    from paper_2604_23826_b200 import DatasetSchema

    s = DatasetSchema.generic(p, False)
    s.identifier_columns = list(ids)
    return s


def plan(n, chunk, precision=0):
    from paper_2604_23826_b200 import PrecisionMode, ReductionPlan, plan_partitions

    return ReductionPlan(plan_partitions(n, chunk), 1, PrecisionMode(precision))


def to_dev(X):
    torch = torch_mod()
    return torch.from_numpy(np.ascontiguousarray(X)).cuda()


def integer_pairs(X):
    """(j,k) packed indices whose columns are integer-valued, and integral column ids."""
    p = X.shape[1]
    integral = [j for j in range(p) if np.all(X[:, j] == np.trunc(X[:, j]))]
    idx = [j * p - j * (j - 1) // 2 + (k - j) for j in integral for k in integral if k >= j]
    return integral, np.array(sorted(idx), dtype=np.int64)


def check_against(got, n, sums, cross, X=None, tol=TOL):
    p = len(sums)
    assert got.n == n
    assert cs_err(got.cross, cross, p) <= tol
    assert sums_err(got.sums, sums, cross, n, p) <= tol
    if X is not None:
        integral, idx = integer_pairs(X)
        if integral:
            assert np.array_equal(bits(got.sums[integral]), bits(sums[integral]))
        if idx.size:
            assert np.array_equal(bits(got.cross[idx]), bits(cross[idx]))


# ----------------------------------------------------------------- known answers
@pytest.mark.parametrize("where", ["host", "device"])
def test_kats(engine, golden, where):
    from paper_2604_23826_b200 import Chunk, NonFiniteError

    for name in ("single_row", "orthogonal"):
        c = golden[name]
        X = np.array(c["rows"], dtype=np.float64)
        vals = X if where == "host" else to_dev(X)
        for flags in (0, 2):
            ss = engine.accumulate_chunk(Chunk(0, X.shape[0], 2, vals), schema(2), flags=flags)
            assert ss.n == c["n"]
            assert np.array_equal(bits(ss.sums), bits(unhex(c["sums"])))
            assert np.array_equal(bits(ss.cross), bits(unhex(c["cross"])))
    bad = np.array([[1.0, 2.0], [3.0, np.inf]])
    vals = bad if where == "host" else to_dev(bad)
    with pytest.raises(NonFiniteError) as ei:
        engine.accumulate_chunk(Chunk(40, 2, 2, vals), schema(2))
    assert (ei.value.row(), ei.value.column()) == (41, 1)
    assert str(ei.value) == golden["nonfinite_chunk"]["error"]["msg"]


def test_empty_chunk_and_schema_mismatch(engine):
    from paper_2604_23826_b200 import Chunk, SchemaMismatchError

    ss = engine.accumulate_chunk(Chunk(0, 0, 3, np.zeros(0)), schema(3))
    assert ss.n == 0 and not ss.sums.any() and not ss.cross.any()
    with pytest.raises(SchemaMismatchError):
        engine.accumulate_chunk(Chunk(0, 1, 2, np.zeros(2)), schema(3))


def test_cauchy_schwarz_random_chunks(engine):
    """test_suffstats.cpp:130-146 on the GPU path."""
    from paper_2604_23826_b200 import Chunk

    rng = np.random.default_rng(77)
    for _ in range(20):
        X = rng.normal(0.0, 3.0, size=(200, 5))
        ss = engine.accumulate_chunk(Chunk(0, 200, 5, X), schema(5))
        S = ss.cross_full()
        for j in range(5):
            for k in range(j + 1, 5):
                assert S[j, k] ** 2 <= S[j, j] * S[k, k] * (1 + 4e-16)


def test_table1_accumulate(engine, oracle, golden):
    from paper_2604_23826_b200 import Chunk, PrecisionMode

    c = golden["table1_seed21"]
    X = oracle.table1_chunk(21, 1, 10000)
    assert sha(X) == c["input_sha256"]
    ref_s, ref_S = unhex(c["sums"]), unhex(c["cross"])
    for vals in (X, to_dev(X)):
        fast = engine.accumulate_chunk(Chunk(0, 10000, 11, vals), schema(11, [0]))
        check_against(fast, 10000, ref_s, ref_S, X)
        exact = engine.accumulate_chunk(Chunk(0, 10000, 11, vals), schema(11, [0]), flags=2)
        assert np.array_equal(bits(exact.sums), bits(ref_s)) and np.array_equal(bits(exact.cross), bits(ref_S))
    c32 = golden["table1_seed21_binary32"]
    f32 = engine.accumulate_chunk(Chunk(0, 10000, 11, X), schema(11, [0]), PrecisionMode.Binary32Diagnostic)
    assert np.array_equal(bits(f32.cross), bits(unhex(c32["cross"])))
    assert np.array_equal(bits(f32.sums), bits(unhex(c32["sums"])))


def test_table1_dataset_every_source(engine, oracle, reference, golden, tmp_path):
    """test_suffstats.cpp:100-128: Table1 seed 5, 20,000 rows, chunk 1024."""
    torch = torch_mod()
    c = golden["table1_seed5_dataset"]
    X = oracle.table1_chunk(5, 1, 20000)
    ref_s, ref_S = unhex(c["sums"]), unhex(c["cross"])
    f = tmp_path / "t5.bin"
    reference.write_binary(str(f), X, 11)
    pinned = torch.from_numpy(X.copy()).pin_memory()
    sources = {"device": to_dev(X), "host": X, "pinned": pinned, "file": str(f)}
    fast = {}
    for name, src in sources.items():
        got = engine.dataset_suffstats(src, schema(11, [0]), plan(20000, 1024))
        check_against(got, 20000, ref_s, ref_S, X)
        fast[name] = got
        exact = engine.dataset_suffstats(src, schema(11, [0]), plan(20000, 1024), flags=2)
        assert np.array_equal(bits(exact.sums), bits(ref_s)) and np.array_equal(bits(exact.cross), bits(ref_S))
    # the fast result is a fixed function of (data, plan): identical for every source
    for name in ("host", "pinned", "file"):
        assert fast[name].bit_equal(fast["device"]), name


GEN_CASES = ["c1_small", "c2_small", "c2_mu0", "ragged_p5", "p24", "p64"]


@pytest.mark.parametrize("name", GEN_CASES)
def test_generated_cases(engine, oracle, reference, golden, name):
    torch = torch_mod()
    c = golden[name]
    g = c["gen"]
    X = oracle.generate(g["kind"], g["seed"], g["mu"], g["n_int"], 0, g["n"], g["p"])
    D = torch.empty((g["n"], g["p"]), dtype=torch.float64, device="cuda")
    engine.generate(D, g["kind"], g["seed"], g["mu"], g["n_int"], 0, g["n"], g["p"])
    assert sha(D.cpu().numpy()) == c["input_sha256"], "GPU generator is not bit-identical to the oracle"
    ids = [0] if g["kind"] == 1 else []
    ref_s, ref_S = unhex(c["sums"]), unhex(c["cross"])
    for flags in (0, 1):  # with and without the per-range shift
        got = engine.dataset_suffstats(D, schema(g["p"], ids), plan(g["n"], g["chunk"]), flags=flags)
        check_against(got, c["n"], ref_s, ref_S, X)
    exact = engine.dataset_suffstats(D, schema(g["p"], ids), plan(g["n"], g["chunk"]), flags=2)
    assert np.array_equal(bits(exact.sums), bits(ref_s)) and np.array_equal(bits(exact.cross), bits(ref_S))
    # downstream (host finalisation of the reference, unchanged) on the GPU SuffStats
    got = engine.dataset_suffstats(D, schema(g["p"], ids), plan(g["n"], g["chunk"]))
    mean, cov, corr = reference.analyze(g["p"], ids, got.n, got.sums, got.cross)
    an = c["analysis"]
    q = mean.size
    iu = np.triu_indices(q)
    rcov = np.zeros((q, q))
    rcov[iu] = unhex(an["cov_upper"])
    rcov = rcov + np.triu(rcov, 1).T
    d = np.sqrt(np.outer(np.diag(rcov), np.diag(rcov)))
    assert np.max(np.abs(cov - rcov) / d) <= TOL
    rcorr = np.zeros((q, q))
    rcorr[iu] = unhex(an["corr_upper"])
    rcorr = rcorr + np.triu(rcorr, 1).T
    assert np.max(np.abs(corr - rcorr)) <= TOL
    for basis, key in ((1, "pca_corr_eigenvalues"), (0, "pca_cov_eigenvalues")):
        ev = reference.run_pca(g["p"], ids, got.n, got.sums, got.cross, basis=basis)
        rev = unhex(c[key])
        assert np.max(np.abs(ev - rev) / np.abs(rev)) <= 1e-10


def test_dataset_nonfinite(engine, oracle, golden, tmp_path, reference):
    from paper_2604_23826_b200 import NonFiniteError, ReductionError

    c = golden["dataset_nonfinite"]
    g = c["gen"]
    X = oracle.generate(g["kind"], g["seed"], g["mu"], g["n_int"], 0, g["n"], g["p"])
    for r, col, kind in c["poison"]:
        X[r, col] = np.inf if kind == "inf" else np.nan
    f = tmp_path / "nf.bin"
    reference.write_binary(str(f), X, 16)
    for src in (to_dev(X), X, str(f)):
        for flags in (0, 2):
            with pytest.raises(ReductionError) as ei:
                engine.dataset_suffstats(src, schema(16), plan(g["n"], g["chunk"]), flags=flags)
            assert ei.value.range_index() == c["error"]["range_index"]
            assert str(ei.value) == c["error"]["msg"]
            assert isinstance(ei.value.cause, NonFiniteError)


def test_overflow_is_not_an_error(engine):
    """Huge finite values overflow the sums to inf without a non-finite input: no error."""
    X = np.full((64, 3), 1e300)
    got = engine.dataset_suffstats(X, schema(3), plan(64, 16))
    assert np.isinf(got.cross[0])


def test_plan_and_file_errors(engine, oracle, reference, tmp_path):
    from paper_2604_23826_b200 import FormatError, IoError, ReductionError, SchemaMismatchError

    X = oracle.generate(0, 1, 1.0, 2, 0, 100, 4)
    with pytest.raises(ValueError, match="partition covers 99 rows"):
        engine.dataset_suffstats(to_dev(X), schema(4), plan(99, 10))
    f = tmp_path / "x.bin"
    reference.write_binary(str(f), X, 4)
    with pytest.raises(ValueError, match="partition covers 99 rows but dataset has 100"):
        engine.dataset_suffstats(str(f), schema(4), plan(99, 10))
    with pytest.raises(ReductionError) as ei:
        engine.dataset_suffstats(str(f), schema(3), plan(100, 10))
    assert isinstance(ei.value.cause, SchemaMismatchError) and ei.value.range_index() == 0
    with pytest.raises(IoError):
        engine.dataset_suffstats(str(tmp_path / "missing.bin"), schema(4), plan(100, 10))
    raw = bytearray(f.read_bytes())
    raw[2] ^= 0xFF
    (tmp_path / "bad.bin").write_bytes(bytes(raw))
    with pytest.raises(FormatError):
        engine.dataset_suffstats(str(tmp_path / "bad.bin"), schema(4), plan(100, 10))
    (tmp_path / "short.bin").write_bytes(f.read_bytes()[:-8])
    with pytest.raises(FormatError):
        engine.dataset_suffstats(str(tmp_path / "short.bin"), schema(4), plan(100, 10))


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
def test_sharded_partials_fold_bit_identical(engine, oracle, W):
    """Row shards per rank (each source holds only its rows) + the rank-ordered fold give the
    single-device result bit-for-bit: the multi-GPU path minus the NCCL copy."""
    import ctypes

    from paper_2604_23826_b200 import _native as N
    from paper_2604_23826_b200 import shard_ranges

    torch = torch_mod()
    n, p, chunk = 300007, 16, 4099
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 42, 1.0, 2, 0, n, p)
    pl = plan(n, chunk)
    whole = engine.dataset_suffstats(D, schema(p), pl)
    R = len(pl.partition.ranges)
    starts = np.array([r.start_row for r in pl.partition.ranges], dtype=np.uint64)
    counts = np.array([r.row_count for r in pl.partition.ranges], dtype=np.uint64)
    E = p + p * (p + 1) // 2
    lmax = (R + W - 1) // W
    stride = 4 + lmax * E
    buf = np.zeros(W * stride)
    lib = N.load()
    for q in range(W):
        f, l = shard_ranges(R, q, W)
        r0 = int(starts[f])
        r1 = int(starts[l - 1] + counts[l - 1])
        shard = D[r0:r1].contiguous()
        src = N.Source(kind=N.SRC_DEVICE, ptr=shard.data_ptr(), first_row=r0, n_rows=r1 - r0)
        out = np.zeros((l - f) * E)
        err = N.Error()
        dp = ctypes.POINTER(ctypes.c_double)
        st = lib.sstat_cuda_range_partials(engine._ctx, ctypes.byref(src), p, starts.ctypes.data, counts.ctypes.data, R,
                                           f, l, 0, 0, out.ctypes.data_as(dp), ctypes.byref(err))
        assert st == 0, err.msg
        buf[q * stride + 4: q * stride + 4 + out.size] = out
    res = np.zeros(E)
    dp = ctypes.POINTER(ctypes.c_double)
    assert lib.sstat_fold_ranges_host(buf.ctypes.data_as(dp), stride, R, W, p, 0, 0, res.ctypes.data_as(dp)) == 0
    assert np.array_equal(bits(res[:p]), bits(whole.sums))
    assert np.array_equal(bits(res[p:]), bits(whole.cross))


@pytest.mark.parametrize("flags", [0, 2])
def test_checkpoint_resume_partials(engine, flags):
    """Checkpoint / resume: per-range partials of a first part of the plan and of the rest,
    computed in separate calls from separate row shards, fold on the host to the bits of one
    dataset_suffstats pass (fast mode and reference order)."""
    from paper_2604_23826_b200 import fold_range_partials

    torch = torch_mod()
    n, p, chunk = 250_003, 24, 7001
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 17, 1.0, 2, 0, n, p)
    pl = plan(n, chunk)
    whole = engine.dataset_suffstats(D, schema(p), pl, flags=flags)
    R = len(pl.partition.ranges)
    k = R // 3
    split_row = pl.partition.ranges[k].start_row
    first = engine.range_partials(D[:split_row].contiguous(), schema(p), pl, 0, k, flags=flags, n_rows=split_row)
    rest = engine.range_partials(D[split_row:].contiguous(), schema(p), pl, k, R, flags=flags, first_row=split_row,
                                 n_rows=n - split_row)
    resumed = fold_range_partials(np.concatenate([first, rest]), schema(p), pl, flags=flags)
    assert resumed.bit_equal(whole)


def test_nccl_world1_identical(oracle):
    """The NCCL exchange path with a communicator of one rank."""
    from paper_2604_23826_b200 import Engine

    torch = torch_mod()
    e = Engine(0)
    uid = Engine.nccl_unique_id()
    e.init_distributed(0, 1, uid)
    n, p = 100000, 16
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    e.generate(D, 0, 3, 1.0, 2, 0, n, p)
    a = e.dataset_suffstats(D, schema(p), plan(n, 8192))
    e2 = Engine(0)
    b = e2.dataset_suffstats(D, schema(p), plan(n, 8192))
    assert a.bit_equal(b)
    e.close()
    e2.close()


def test_streaming_small_slots_bit_identical(engine, oracle):
    """Host sources stream through the staging ring; tiny slots force many chunks."""
    from paper_2604_23826_b200 import Engine

    torch = torch_mod()
    n, p = 1 << 20, 16
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 5, 1.0, 2, 0, n, p)
    H = D.cpu()
    dev = engine.dataset_suffstats(D, schema(p), plan(n, 100003))
    e = Engine(0)
    e.set_staging(3, 1 << 20)
    assert e.dataset_suffstats(H.numpy(), schema(p), plan(n, 100003)).bit_equal(dev)
    assert e.dataset_suffstats(H.pin_memory(), schema(p), plan(n, 100003)).bit_equal(dev)
    e.close()


@pytest.mark.parametrize("threads", [1, 3, 16])
def test_feeder_threads_bit_identical(engine, tmp_path, threads):
    """The host feeder (parallel pread / memcpy of row blocks into the staging slots) gives
    the same bits for any thread count, for pageable and file sources, including slots
    that do not split evenly and a ragged last chunk."""
    from paper_2604_23826_b200 import Engine

    torch = torch_mod()
    n, p = 3_000_017, 13
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 9, 0.0, 2, 0, n, p)
    H = D.cpu().numpy()
    path = tmp_path / "feed.bin"
    hdr = bytearray(64)
    hdr[0:8] = b"SSTATBIN"
    hdr[8:12] = (1).to_bytes(4, "little")
    hdr[12:20] = n.to_bytes(8, "little")
    hdr[20:24] = p.to_bytes(4, "little")
    with open(path, "wb") as f:
        f.write(hdr)
        H.tofile(f)
    dev = engine.dataset_suffstats(D, schema(p), plan(n, 1 << 18))
    e = Engine(0)
    e.set_staging(3, 40 << 20)
    e.set_host_threads(threads)
    assert e.dataset_suffstats(H, schema(p), plan(n, 1 << 18)).bit_equal(dev)
    assert e.dataset_suffstats(str(path), schema(p), plan(n, 1 << 18)).bit_equal(dev)
    e.close()


def test_c1_full_size(engine, oracle):
    """Config 1: 1e6 x (8 + ID), the ID column excluded downstream.  The reference's own
    sequential sum of id^2 (3.3e17 > 2^53) is 1.1e-12 off the true value, so entries are
    held to the extended-precision truth; the reference is held to its own error + 1e-12."""
    torch = torch_mod()
    n, p = 1_000_000, 9
    X = oracle.generate(1, 42, 1.0, 0, 0, n, p)
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 1, 42, 1.0, 0, 0, n, p)
    assert np.array_equal(bits(D.cpu().numpy()), bits(X))
    s, c = oracle.plan_partitions(n, 1 << 20)
    want = oracle.run_reduction(X, p, s, c, 8)
    got = engine.dataset_suffstats(D, schema(p, [0]), plan(n, 1 << 20))
    assert got.sums[0] == want[1][0] == n * (n + 1) / 2  # identifier sum, exact
    ts, tS = truth_suffstats(X)
    assert tS[0] == float(n * (n + 1) * (2 * n + 1) // 6)
    check_against(got, n, ts, tS)
    ref_err = cs_err(want[2], tS, p)
    assert cs_err(got.cross, want[2], p) <= ref_err + TOL


def test_c2_full_size_properties(engine):
    """Config 2 at full size (1e8 x 16, HBM-resident): fast vs the reference-order mode
    (bit-identical to the reference by construction) — integer block bit-exact, the rest
    within tolerance; covariance near the generator's known tridiagonal Sigma."""
    torch = torch_mod()
    n, p = 100_000_000, 16
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 0, 42, 1.0, 2, 0, n, p)
    pl = plan(n, 1 << 20)
    fast = engine.dataset_suffstats(D, schema(p), pl)
    exact = engine.dataset_suffstats(D, schema(p), pl, flags=2)
    assert fast.n == exact.n == n
    idx = [0, 1, p]  # (0,0), (0,1), (1,1)
    assert np.array_equal(bits(fast.cross[idx]), bits(exact.cross[idx]))
    assert np.array_equal(bits(fast.sums[:2]), bits(exact.sums[:2]))
    assert cs_err(fast.cross, exact.cross, p) <= TOL
    assert sums_err(fast.sums, exact.sums, exact.cross, n, p) <= TOL
    mu = fast.sums / n
    cov = fast.cross_full() / n - np.outer(mu, mu)
    g = cov[2:, 2:]
    want = np.diag([1.0] + [1.25] * 13) + np.diag([0.5] * 13, 1) + np.diag([0.5] * 13, -1)
    assert np.max(np.abs(g - want)) < 2e-3
    del D
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["wide_p80", "wide_p256"])
def test_wide_p_cases(engine, oracle, reference, golden, name):
    """K2 (p > 64, DMMA SYRK) against the reference: sums bit-pinned golden, X^T X via the
    oracle (pinned to the reference by SHA-256), eigenvalues via the reference's run_pca."""
    torch = torch_mod()
    c = golden[name]
    g = c["gen"]
    p = g["p"]
    X = oracle.generate(g["kind"], g["seed"], g["mu"], g["n_int"], 0, g["n"], p)
    assert sha(X) == c["input_sha256"]
    s0, c0 = oracle.plan_partitions(g["n"], g["chunk"])
    wn, ws, wS = oracle.run_reduction(X, p, s0, c0, 8)
    assert sha(wS) == c["cross_sha256"], "oracle X^T X no longer matches the reference"
    D = to_dev(X)
    for flags in (0, 1):
        got = engine.dataset_suffstats(D, schema(p), plan(g["n"], g["chunk"]), flags=flags)
        check_against(got, wn, unhex(c["sums"]), wS)
    exact = engine.dataset_suffstats(D, schema(p), plan(g["n"], g["chunk"]), flags=2)
    assert np.array_equal(bits(exact.cross), bits(wS)) and np.array_equal(bits(exact.sums), bits(unhex(c["sums"])))
    got = engine.dataset_suffstats(D, schema(p), plan(g["n"], g["chunk"]))
    for basis, key in ((1, "pca_corr_eigenvalues"), (0, "pca_cov_eigenvalues")):
        ev = reference.run_pca(p, [], got.n, got.sums, got.cross, basis=basis)
        rev = unhex(c[key])
        assert np.max(np.abs(ev - rev) / np.abs(rev)) <= 1e-10
    # host-streamed source gives the same bits
    assert engine.dataset_suffstats(X, schema(p), plan(g["n"], g["chunk"])).bit_equal(got)


@pytest.mark.parametrize("p", [65, 72, 97, 128, 130, 200, 256, 300, 513, 1024])
def test_wide_p_shapes_vs_truth(engine, oracle, p):
    """Odd / ragged wide p (masked column blocks, 8-byte staging for odd p), ragged ranges;
    p spans every cluster shape (2..9 CTAs of 4 warps, clusters of 8-warp CTAs, several
    clusters per tile) and stage height (16 / 8 / 4 rows)."""
    rng = np.random.default_rng(p)
    n = 70001 if p <= 256 else 9001
    X = rng.normal(1.0, 1.0, size=(n, p))
    X[:, 0] = rng.integers(1, 100, size=n)
    X[:, 1] = rng.integers(1, 100, size=n)
    ts, tS = truth_suffstats(X)
    got = engine.dataset_suffstats(to_dev(X), schema(p), plan(n, 33333))
    check_against(got, n, ts, tS)
    assert np.array_equal(bits(got.cross[[0, 1, p]]), bits(tS[[0, 1, p]]))  # integer block exact


@pytest.mark.parametrize("p", [65, 73, 81, 89, 97, 105, 113, 121])
def test_k1w_extra_column_widths(engine, p, monkeypatch):
    """p = 8 NB + 1 in K1w: NB block rows plus the last column by DFMA (part 0 of each row
    group) against the 80-bit truth, integer block bit-exact, ragged tiles and ranges; the
    (NB + 1)-block-row split (SSTAT_K1W_NO_X1) agrees within the same tolerance."""
    rng = np.random.default_rng(1000 + p)
    n = 70001
    X = rng.normal(-0.5, 1.5, size=(n, p))
    X[:, 0] = rng.integers(1, 100, size=n)
    X[:, p - 1] = rng.integers(1, 100, size=n)  # the extra column itself integer-valued
    ts, tS = truth_suffstats(X)
    D = to_dev(X)
    got = engine.dataset_suffstats(D, schema(p), plan(n, 33331))
    check_against(got, n, ts, tS)
    last = p - 1
    exact = [0, last, last * p - last * (last - 1) // 2]  # Σx0², Σx0·x_last, Σx_last² (SymPacked)
    assert np.array_equal(bits(got.cross[exact]), bits(tS[exact]))
    assert np.array_equal(bits(got.sums[[0, last]]), bits(ts[[0, last]]))
    monkeypatch.setenv("SSTAT_K1W_NO_X1", "1")
    check_against(engine.dataset_suffstats(D, schema(p), plan(n, 33331)), n, ts, tS)


@pytest.mark.parametrize("p", [65, 72, 81, 92, 96, 97, 104, 128])
def test_k1w_load_depth_bit_identical(engine, p, monkeypatch):
    """K1w's loads in flight (U = 2 / 3 / 4 k-steps, SSTAT_K1W_U) only batch the loads: each
    warp accumulates the same k-steps in the same order, so every depth gives the same bits."""
    torch = torch_mod()
    n = 90001
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 2, 5, 1.0, 0, 0, n, p)
    pl = plan(n, 40009)
    base = engine.dataset_suffstats(D, schema(p), pl)
    for u in ("2", "3", "4"):
        with monkeypatch.context() as m:
            m.setenv("SSTAT_K1W_U", u)
            assert engine.dataset_suffstats(D, schema(p), pl).bit_equal(base), u


def test_every_p_up_to_72(engine):
    """Every width through K1's template instances (column blocks 1..8, vector and scalar
    loads) and across the K1 -> K2 switch at p = 64 / 65, ragged tiles and ranges: the
    80-bit truth within tolerance, integer columns bit-exact."""
    rng = np.random.default_rng(2024)
    for p in range(1, 73):
        n = 2003 + 37 * p
        X = rng.normal(0.5, 2.0, size=(n, p))
        X[:, : min(2, p)] = rng.integers(-50, 100, size=(n, min(2, p)))
        ts, tS = truth_suffstats(X)
        got = engine.dataset_suffstats(to_dev(X), schema(p), plan(n, 977))
        check_against(got, n, ts, tS, X)


def test_buffer_growth_sequence():
    """One context through growing and shrinking widths, a non-finite call in between: the
    error header and range flags are reset whenever a buffer is reallocated (a new allocation
    can reuse the old address with fresh, zeroed pages), so clean calls never report stale
    failures and the failing call reports the right cell."""
    from paper_2604_23826_b200 import Engine, ReductionError

    torch = torch_mod()
    e = Engine(0)
    rng = np.random.default_rng(11)
    for p, bad in ((16, None), (700, None), (9, (5, 3)), (1024, None), (16, None), (1500, None), (64, (70, 63))):
        n = 3000
        X = rng.normal(0.0, 1.0, size=(n, p))
        if bad:
            X[bad] = np.nan
            with pytest.raises(ReductionError, match=f"row {bad[0]}, column {bad[1]}"):
                e.dataset_suffstats(to_dev(X), schema(p), plan(n, 1000))
        else:
            ts, tS = truth_suffstats(X) if p <= 256 else (None, None)
            got = e.dataset_suffstats(to_dev(X), schema(p), plan(n, 1000))
            assert got.n == n and np.all(np.isfinite(got.cross))
            if ts is not None:
                check_against(got, n, ts, tS)
    e.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("p", [9, 16, 32, 256])
def test_misaligned_device_rows(engine, p):
    """A device pointer that is only 8-byte aligned (a view one double into a buffer) takes
    the scalar-load / 8-byte cp.async paths and gives the same bits as an aligned copy (in
    reference-order mode too: cp.async staging vs the TMA ring)."""
    torch = torch_mod()
    n = 50_001
    buf = torch.empty(n * p + 1, dtype=torch.float64, device="cuda")
    D = buf[1:].view(n, p)
    assert D.data_ptr() % 16 == 8
    engine.generate(D, 2, 3, 0.25, 0, 0, n, p)
    A = D.clone()
    assert A.data_ptr() % 16 == 0
    assert engine.dataset_suffstats(D, schema(p), plan(n, 9999)).bit_equal(
        engine.dataset_suffstats(A, schema(p), plan(n, 9999)))
    if p <= 64:  # reference order: the cp.async-staged kernel (misaligned) vs the TMA ring (aligned)
        assert engine.dataset_suffstats(D, schema(p), plan(n, 9998), flags=2).bit_equal(
            engine.dataset_suffstats(A, schema(p), plan(n, 9998), flags=2))


def test_widest_fast_path_and_limit(engine, oracle):
    """p = 2048 (K2's widest: 4-row stages, many clusters per tile) against the oracle; p = 2049
    is refused by the fast path with UNSUPPORTED and served by reference-order mode, bit-exact."""
    from paper_2604_23826_b200 import DeviceError

    rng = np.random.default_rng(7)
    n, p = 1500, 2048
    X = rng.normal(0.0, 1.0, size=(n, p))
    s0, c0 = oracle.plan_partitions(n, 700)
    wn, ws, wS = oracle.run_reduction(X, p, s0, c0, 1)
    got = engine.dataset_suffstats(to_dev(X), schema(p), plan(n, 700))
    check_against(got, wn, ws, wS)
    n, p = 40, 2049
    X = rng.normal(0.0, 1.0, size=(n, p))
    with pytest.raises(DeviceError, match="2048"):
        engine.dataset_suffstats(to_dev(X), schema(p), plan(n, 16))
    s0, c0 = oracle.plan_partitions(n, 16)
    wn, ws, wS = oracle.run_reduction(X, p, s0, c0, 1)
    exact = engine.dataset_suffstats(to_dev(X), schema(p), plan(n, 16), flags=2)
    assert exact.n == wn and np.array_equal(bits(exact.cross), bits(wS)) and np.array_equal(bits(exact.sums), bits(ws))


@pytest.mark.parametrize("p", [96, 256, 259, 520])
def test_wide_p_schedule_invariant(engine, p, monkeypatch):
    """K2's result is a fixed function of the tile: 4- or 8-warp groups, with or without the
    cluster multicast, with or without the cluster-less side launch claiming tiles
    dynamically, 2-, 3- or 4-block rectangles, and the 12-consumer-warp k_widep_wg give the
    same bits."""
    torch = torch_mod()
    monkeypatch.setenv("SSTAT_SPLITP", "0")  # K2 itself at every p (K1w takes 64 < p <= 128 by default)
    n = 100003 if p <= 256 else 40001
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 2, 7, 1.5, 0, 0, n, p)
    pl = plan(n, 30011)
    base = engine.dataset_suffstats(D, schema(p), pl)
    for env in ({"SSTAT_WIDEP_CONSUMERS": "8"}, {"SSTAT_WIDEP_CONSUMERS": "4"}, {"SSTAT_WIDEP_NOCLUSTER": "1"},
                {"SSTAT_WIDEP_SPARE": "0"}, {"SSTAT_WIDEP_R": "2"}, {"SSTAT_WIDEP_R": "3"}, {"SSTAT_WIDEP_R": "4"},
                {"SSTAT_WIDEP_WG": "1"}, {"SSTAT_WIDEP_WG": "1", "SSTAT_WIDEP_R": "3"},
                {"SSTAT_WIDEP_WG": "1", "SSTAT_WIDEP_SPARE": "0"}, {"SSTAT_WIDEP_WG": "1", "SSTAT_WIDEP_NOCLUSTER": "1"}):
        with monkeypatch.context() as m:
            for k, v in env.items():
                m.setenv(k, v)
            assert engine.dataset_suffstats(D, schema(p), pl).bit_equal(base), env
    del D
    torch.cuda.empty_cache()


def test_c5_scale_wide(engine):
    """Config 5 shape (p = 256) at 4e6 rows on one GPU (the full 1e8 x 256 = 204.8 GB needs
    two B200s): fast vs reference-order mode."""
    torch = torch_mod()
    n, p = 4_000_000, 256
    D = torch.empty((n, p), dtype=torch.float64, device="cuda")
    engine.generate(D, 2, 19, 1.0, 0, 0, n, p)
    pl = plan(n, 1 << 20)
    fast = engine.dataset_suffstats(D, schema(p), pl)
    exact = engine.dataset_suffstats(D, schema(p), pl, flags=2)
    assert cs_err(fast.cross, exact.cross, p) <= TOL
    assert sums_err(fast.sums, exact.sums, exact.cross, n, p) <= TOL
    del D
    torch.cuda.empty_cache()


def test_concurrent_engines_threads():
    """Two contexts driven from two host threads at once (K1, K1w and K2 widths, device and
    host sources, K2's shared plan cache and side stream) give the same bits as one at a time."""
    import threading

    from paper_2604_23826_b200 import Engine

    torch = torch_mod()
    cases = [(16, 200_003), (256, 60_001), (104, 50_001), (72, 40_003)]
    data = []
    e0 = Engine(0)
    for p, n in cases:
        D = torch.empty((n, p), dtype=torch.float64, device="cuda")
        e0.generate(D, 2, 31, 0.5, 0, 0, n, p)
        data.append((D, p, n))
    want = [e0.dataset_suffstats(D, schema(p), plan(n, 30_011)) for D, p, n in data]
    got = {}
    errors = []

    def worker(tid):
        try:
            e = Engine(0)
            for rep in range(3):
                for i, (D, p, n) in enumerate(data):
                    src = D if (i + tid + rep) % 2 == 0 else D.cpu().numpy()
                    got[(tid, rep, i)] = e.dataset_suffstats(src, schema(p), plan(n, 30_011))
            e.close()
        except Exception as ex:  # pragma: no cover - reported below
            errors.append(ex)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (tid, rep, i), ss in got.items():
        assert ss.bit_equal(want[i]), (tid, rep, i)
    e0.close()
