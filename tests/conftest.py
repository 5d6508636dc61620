"""Shared fixtures.  The oracle (oracle/) is used here only as the checker."""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], dtype=np.float64)


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle

    return Oracle()


@pytest.fixture(scope="session")
def reference():
    """The unmodified reference library; built here, shipped prebuilt to the GPU box."""
    from oracle.oracle import REF_SO, REF_SRC, Reference

    if not os.path.exists(REF_SO) and not os.path.isdir(REF_SRC):
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return Reference()


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def engine():
    if not gpu_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_2604_23826_b200 import Engine

    e = Engine(0)
    yield e
    e.close()


def cs_err(got_cross: np.ndarray, ref_cross: np.ndarray, p: int) -> float:
    """max |dS_jk| / sqrt(S_jj S_kk) over the packed triangle (Cauchy-Schwarz normalised)."""
    iu = np.triu_indices(p)
    diag = np.array([ref_cross[j * p - j * (j - 1) // 2] for j in range(p)])
    scale = np.sqrt(np.abs(diag[iu[0]] * diag[iu[1]]))
    scale[scale == 0] = 1.0
    return float(np.max(np.abs(got_cross - ref_cross) / scale))


def sums_err(got_sums, ref_sums, ref_cross, n, p) -> float:
    """max |ds_j| / sqrt(n S_jj)."""
    diag = np.array([ref_cross[j * p - j * (j - 1) // 2] for j in range(p)])
    scale = np.sqrt(np.abs(n * diag))
    scale[scale == 0] = 1.0
    return float(np.max(np.abs(got_sums - ref_sums) / scale))


def truth_suffstats(X: np.ndarray):
    """Sums and packed X^T X accumulated in extended precision (80-bit long double, pairwise):
    error ~1e-19 relative, far below the 1e-12 bar — the yardstick where the reference's own
    sequential binary64 sums exceed the bar (e.g. the identifier's sum of squares at 1e6 rows)."""
    L = X.astype(np.longdouble)
    p = X.shape[1]
    sums = L.sum(axis=0)
    cross = [np.sum(L[:, j] * L[:, k]) for j in range(p) for k in range(j, p)]
    return sums.astype(np.float64), np.array(cross, dtype=np.longdouble).astype(np.float64)
