"""A few cfg-5 fresh gathers at n^3 with run-time options (for ncu A/B):
python scripts/fresh_once.py n [OPT=V ...]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402

n = int(sys.argv[1])
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in sys.argv[2:]}
a = drivers.alloc("wave3d_r4", n)
drivers.init_static("wave3d_r4", a, n, 0)
drivers.regen_step(a["u_1"], a["u_b"], n, 0, 0, 4)
with api.options(**opts):
    for _ in range(3):
        api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a)
torch.cuda.synchronize()
print("ok")
