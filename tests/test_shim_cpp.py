"""Runs the C++ parity harness (tests/cpp/shim_parity.cpp): this repo's
reference-signature C++ API next to the unmodified reference library in one
process, every application config x every strategy, bitwise."""
import os
import subprocess

import pytest

from gspmm_testutil import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "shim_parity")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="shim_parity not built (needs /root/reference)")
def test_cpp_shim_matches_reference_library():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 failures" in r.stdout
