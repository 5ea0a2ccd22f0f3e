"""One host-API gather adjoint call on oracle-style inputs (developer aid):
    python scripts/one_call.py <family> <n>"""
import sys
import numpy as np
sys.path.insert(0, ".")
from tests import inputs as gen
from paper_1907_02818_b200 import api
name, n = sys.argv[1], int(sys.argv[2])
scalars, grids, adjs = gen.family_inputs(name, n, seed=n, accumulate=True)
r = api.run_program(name, n, scalars, grids, adjs, dtype="f32")
print("ok", float(np.abs(r["c_b"]).sum()))
