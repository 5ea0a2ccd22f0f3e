"""Radius-1 fp32 gather: fp32 vs fp64 accumulation (R1_FP64ACC), kernel time at
cfg 2's 512^3 (accumulating entry and the carried sweep's fresh-u2 entry)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402
from scripts.quick_time import time_it  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
fam = "wave3d_c"
a = drivers.alloc(fam, n)
drivers.init_static(fam, a, n, 0)
drivers.regen_state(a["u_1"], n, 0, 0, 1)
drivers.regen_seed(a["u_b"], n, 1, 0)
bpp = 36
for acc in (0, 1):
    with api.options(R1_FP64ACC=acc):
        t1 = time_it(lambda: api.adjoint(fam, n, {"D": 0.1}, a), iters=30)
        t2 = time_it(lambda: api.adjoint_fresh_u2(fam, n, {"D": 0.1}, a), iters=30)
    print(f"R1_FP64ACC={acc} n={n}: adjoint {t1:.3f} ms ({bpp * n**3 / t1 / 1e6:.0f} GB/s), "
          f"fresh_u2 {t2:.3f} ms ({(bpp - 4) * n**3 / t2 / 1e6:.0f} GB/s)")
