"""Runs the reference user's program (tests/native/adapter_vs_reference.cpp,
built as oracle/_ref/adapter_check from the real reference headers in the
build container): the reference's hdivmg::MGPreconditioner and the drop-in
hpmg::MGPreconditioner side by side in one process on identical inputs:
operator, rhs, apply, pcg(A, M, b, x) with the reference's own generic
Krylov loop and the device preconditioner, the device-resident pcg, and
uzawa_solve (counts +-1, velocity <= 1e-9)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.mark.skipif(not os.path.exists(BIN), reason="adapter_check not built (needs the reference tree at build)")
def test_adapter_against_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "all checks passed" in r.stdout
