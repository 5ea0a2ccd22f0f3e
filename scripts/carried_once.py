"""A few cfg-2 carried-sweep gathers (wave3d_c_b_fresh_u2_f32, the fp64-
arithmetic radius-1 kernel) at 512^3 for ncu; developer aid.
python scripts/carried_once.py [R1_FP64ACC=0|1]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402

acc = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n, fam = 512, "wave3d_c"
a = drivers.alloc(fam, n)
drivers.init_static(fam, a, n, 0)
drivers.regen_state(a["u_1"], n, 0, 0, 1)
drivers.regen_seed(a["u_b"], n, 1, 0)
with api.options(R1_FP64ACC=acc):
    for _ in range(3):
        api.adjoint_fresh_u2(fam, n, {"D": 0.1}, a)
        api.adjoint(fam, n, {"D": 0.1}, a)
torch.cuda.synchronize()
print("ok")
