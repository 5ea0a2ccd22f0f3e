"""The INTEGRATION.md reference-side binding, compiled against the UNMODIFIED
reference headers and library (oracle/ref/b200_binding.cpp, linked into
oracle/_ref/ref_harness): run_program_b200(p, env) on the reference's own
Problem / Env / DenseGrid must equal the reference's run_program(p, env)
(interp.hpp:59) at the reference's 1e-12 oracle-equivalence bound.
"""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle
from tests.test_oracle_pins import _golden_cases, load_golden

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1907_02818_b200", "libstencilgrad_b200.so")
FAMS = ("wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4")


@pytest.mark.parametrize("case", [c for c in _golden_cases() if c.rsplit("_n", 1)[0] in FAMS])
def test_reference_binding_matches_reference_run_program(case):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref/ref_harness not built (needs /root/reference at build time)")
    name, n, f, scalars, grids, adjs, _ = load_golden(case)
    with tempfile.TemporaryDirectory() as td:
        for k, v in {**grids, **adjs}.items():
            np.ascontiguousarray(v, dtype=np.float64).tofile(os.path.join(td, k + ".f64"))
        r = subprocess.run([oracle.ref_harness_path(), "b200", oracle.spec_path(name), str(n), td,
                            *[f"{k}={v!r}" for k, v in scalars.items()]],
                           capture_output=True, text=True, env=dict(os.environ, SGB_LIB=LIB),
                           timeout=120)
    assert r.returncode in (0, 1), r.stderr
    rep = json.loads(r.stdout)
    assert rep["max_rel_err"] <= 1e-12, rep
