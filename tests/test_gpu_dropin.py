"""C++ drop-in: the reference engine and hyperanf_b200::NfEngine
(include/hyperanf_b200/engine.hpp over libhanf.so) on the same
hyperanf::Graph objects, lockstep bit-exact (tests/cpp/dropin_test.cpp,
built into oracle/_ref/ by oracle/Makefile)."""
from __future__ import annotations

import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="dropin_test not built (needs the reference headers)")
def test_cpp_dropin_lockstep():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
