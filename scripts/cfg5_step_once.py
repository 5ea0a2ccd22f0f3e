"""A few cfg-5 reverse steps at 1024^3 (regenerate u_1 / u_b, fused fresh
gather) for ncu: the generator and MODE-4 radius-4 kernels the bench times.
python scripts/cfg5_step_once.py [n]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
a = drivers.alloc("wave3d_r4", n)
drivers.init_static("wave3d_r4", a, n, 0)
for t in range(3):
    drivers.regen_step(a["u_1"], a["u_b"], n, t, 0, 4)
    api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a)
torch.cuda.synchronize()
print("ok")
