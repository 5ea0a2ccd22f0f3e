"""Scratch timing of the fp64 3D gather adjoints at full size (developer aid)."""
import sys, torch
sys.path.insert(0, ".")
from paper_1907_02818_b200 import api
from scripts.quick_time import time_it
for fam, n, sc, bpp in [("wave3d_r4", 768, {"D": 0.01}, 56), ("wave3d_c", 512, {"D": 0.1}, 72)]:
    arrays = {nm: torch.randn((n, n, n), dtype=torch.float64, device="cuda") for nm in api.array_params(fam, "adjoint")}
    ms = time_it(lambda: api.adjoint(fam, n, sc, arrays), iters=5, warm=2)
    print(fam, n, "f64 adjoint", round(ms, 3), "ms", round(n**3 * bpp / ms / 1e6), "GB/s")
