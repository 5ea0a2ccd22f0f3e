"""Scratch timing of the companion kernels (primal, box_axpy) at full size."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api  # noqa: E402
from scripts.quick_time import time_it  # noqa: E402

# algorithmic bytes/pt: arrays read + written once (wave3d_c is a '+=' primal: u read too)
for fam, n, bpp in [("wave3d_r4", 768, 16), ("wave3d_c", 512, 20), ("wave1d", 1 << 24, 32),
                    ("burgers2d", 8192, 16)]:
    a = bench.gen_inputs(api, torch, fam, n)
    dt = a[next(iter(a))].dtype
    shape = a[next(iter(a))].shape
    prim = {nm: torch.randn(shape, dtype=dt, device="cuda") for nm in
            api.array_params(fam, "primal")}
    sc = bench.CONFIGS[{"wave3d_r4": "4", "wave3d_c": "2", "wave1d": "1", "burgers2d": "3"}[fam]][4]
    ms = time_it(lambda: api.primal(fam, n, sc, prim))
    pts = n ** (3 if fam.startswith("wave3d") else 2 if fam == "burgers2d" else 1)
    print(f"{fam:10s} primal {ms:.3f} ms  {pts * bpp / ms / 1e6:.0f} GB/s  ({bpp} B/pt)")
a = torch.randn(768, 768, 768, device="cuda")
b = torch.randn_like(a)
ms = time_it(lambda: api.box_axpy(a, b, -1.0, 768, 4, 763))
print(f"box_axpy 768^3 {ms:.3f} ms {768 ** 3 * 12 / ms / 1e6:.0f} GB/s")
