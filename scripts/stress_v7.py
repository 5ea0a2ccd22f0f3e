"""Repeat the radius-4 gather many times on the same inputs and count runs that
differ from the first (developer aid for races):
    python scripts/stress_v7.py wave3d_r4 <n> <reps>"""
import os, sys
import numpy as np
sys.path.insert(0, ".")
import torch
from tests import inputs as gen
from paper_1907_02818_b200 import api
name, n, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
scalars, grids, adjs = gen.family_inputs(name, n, seed=n, accumulate=True)
dev = {k: torch.from_numpy(v.astype(np.float32)).cuda() for k, v in {**grids, **adjs}.items()}
# reference: generic per-point kernel via slab entry with n not TMA? use full-grid default (v5/v1)
ref = {k: v.clone() for k, v in dev.items()}
api.adjoint(name, n, scalars, ref)
torch.cuda.synchronize()
nbad_runs = 0
for r in range(reps):
    out = {k: v.clone() for k, v in dev.items()}
    api.adjoint(name, n, scalars, out)
    torch.cuda.synchronize()
    for k in adjs:
        d = (out[k] - ref[k]).abs()
        if float(d.max()) > 1e-5:
            bad = torch.nonzero(d > 1e-5)
            nbad_runs += 1
            print(r, k, "bad", bad.shape[0], "planes", bad[:, 0].unique()[:10].tolist(),
                  "rows", bad[:, 1].unique()[:10].tolist(), "cols", bad[:, 2].unique()[:8].tolist())
print(name, n, "runs with errors:", nbad_runs, "of", reps)
