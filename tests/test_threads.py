"""Host-thread safety of the C ABI (tests/cpp/test_threads.cpp): T threads per
visible device make their first library calls at the same moment, each on
its own stream and buffers, and match one serial call bitwise."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1907_02818_b200")


def _build(out):
    from paper_1907_02818_b200 import build as b
    b.build()
    cmd = ["g++", "-std=c++17", "-O2", "-pthread",
           os.path.join(ROOT, "tests", "cpp", "test_threads.cpp"),
           "-I" + os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L" + LIBDIR,
           "-lstencilgrad_b200", "-L/usr/local/cuda/lib64", "-lcudart",
           "-Wl,-rpath," + LIBDIR, "-Wl,-rpath,/usr/local/cuda/lib64", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def test_threads_caller_builds(tmp_path):
    assert os.path.exists(_build(str(tmp_path / "test_threads")))


@pytest.mark.gpu
@pytest.mark.parametrize("threads,iters", [(8, 3), (16, 2)])
def test_concurrent_first_calls_match_serial(tmp_path, threads, iters):
    exe = _build(str(tmp_path / "test_threads"))
    r = subprocess.run([exe, str(threads), str(iters)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failures" in r.stdout, r.stdout
