"""Runs the C++ drop-in API test binary (tests/cpp/test_api.cpp) on the GPU:
the reference-style kernel and solver checks through blockkrylov/*.hpp ->
include/bkg.h -> libbkgpu.so, in exact and fast numerics."""
import os
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "bin", "test_api")


def test_cpp_binary_is_built():
    assert os.path.exists(BIN), "build with __graft_entry__.build()"


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_cpp_dropin_api(mode):
    r = subprocess.run([BIN, mode], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout
