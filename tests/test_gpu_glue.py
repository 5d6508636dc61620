"""The reference's own C++ library driven through integration/sstat_cuda_glue.hpp on the GPU
(oracle/glue_test.cpp): stage-6 bit-exactness, finalisation tolerances, run_reduction
plugin, error mapping, sidecar round trip."""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

GLUE = os.path.join(ROOT, "oracle", "_ref", "glue_test")


def test_reference_driver_through_glue():
    if not os.path.exists(GLUE):
        pytest.fail("oracle/_ref/glue_test not built (run __graft_entry__.build() where /root/reference exists)")
    r = subprocess.run([GLUE], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr
    assert "glue_test: OK" in r.stdout
