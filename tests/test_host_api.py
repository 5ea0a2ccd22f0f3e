"""The C++ host API (include/stencilgrad_b200.hpp) -- the reference's
interp.hpp entry points over the C ABI -- built with g++ against the in-tree
library and run (tests/cpp/test_host_api.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1907_02818_b200")
ORACLE = os.path.join(ROOT, "oracle")


def _build(out):
    from paper_1907_02818_b200 import build as b
    b.build()
    cmd = ["g++", "-std=c++17", "-O2", os.path.join(ROOT, "tests", "cpp", "test_host_api.cpp"),
           "-I" + os.path.join(ROOT, "include"), "-I" + ORACLE, "-L" + LIBDIR,
           "-lstencilgrad_b200", "-L" + ORACLE, "-loracle", "-Wl,-rpath," + LIBDIR,
           "-Wl,-rpath," + ORACLE, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_host_api_builds_and_links(tmp_path):
    """CPU: the C++ API header compiles and the test links against the
    library (the symbols exist); running needs a GPU."""
    from oracle import oracle
    oracle.build()
    assert os.path.exists(_build(str(tmp_path / "test_host_api")))


@pytest.mark.gpu
def test_host_api_matches_oracle(tmp_path):
    from oracle import oracle
    oracle.build()
    exe = _build(str(tmp_path / "test_host_api"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
