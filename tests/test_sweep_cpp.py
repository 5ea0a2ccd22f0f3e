"""The host-state sweeps (sgb_plan_sweep_*) called from plain C++ over the C
ABI, as INTEGRATION.md shows them (tests/cpp/test_sweep.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1907_02818_b200")


def _build(out):
    from paper_1907_02818_b200 import build as b
    b.build()
    cmd = ["g++", "-std=c++17", "-O2", os.path.join(ROOT, "tests", "cpp", "test_sweep.cpp"),
           "-I" + os.path.join(ROOT, "include"), "-L" + LIBDIR, "-lstencilgrad_b200",
           "-Wl,-rpath," + LIBDIR, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_sweep_cpp_builds_and_links(tmp_path):
    assert os.path.exists(_build(str(tmp_path / "test_sweep")))


@pytest.mark.gpu
def test_sweep_cpp_matches_per_step_calls(tmp_path):
    exe = _build(str(tmp_path / "test_sweep"))
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
