"""The reference's own acceptance gate (tests/acceptance.cpp, unmodified),
linked against the B200 drop-in shim instead of src/big_means.cpp
(tools/dropin/Makefile).  Criterion 3 checks big_means(s=m) on the GPU
against the reference's CPU kmeans bit for bit; 2 checks monotone traces;
9 checks determinism across reference worker counts."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "dropin", "_build", "acceptance_b200")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in binary not built (needs /root/reference)")
@pytest.mark.parametrize("criterion", [2, 3, 9])
def test_reference_acceptance_through_dropin(criterion):
    r = subprocess.run([BIN, str(criterion)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "PASS" in r.stdout, r.stdout + r.stderr
