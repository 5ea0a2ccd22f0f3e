"""fp64 radius-4 gathers (fresh MODE 4 and accumulating) and the fp64 pair
generator across grid sizes, kernel-alone CUDA-event medians (developer aid):
    python scripts/f64_sizes.py [n ...]
Prints ms and algorithmic GB/s (fresh 48 B/pt, accumulating 56, generator 16)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402
from scripts.quick_time import time_it  # noqa: E402

sizes = [int(x) for x in sys.argv[1:]] or [768, 1000, 1024]
for n in sizes:
    a = {nm: torch.zeros((n, n, n), dtype=torch.float64, device="cuda")
         for nm in api.array_params("wave3d_r4", "adjoint")}
    a["c"].uniform_(1.5, 4.5)
    drivers.regen_step(a["u_1"], a["u_b"], n, 0, 0, 4)
    pts = float(n) ** 3
    g = time_it(lambda: drivers.regen_step(a["u_1"], a["u_b"], n, 1, 0, 4), iters=10)
    f = time_it(lambda: api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a), iters=10)
    c = time_it(lambda: api.adjoint("wave3d_r4", n, {"D": 0.01}, a), iters=10)
    print(f"n={n}: pair generator {g:.3f} ms ({16 * pts / g / 1e6:.0f} GB/s), "
          f"fresh gather {f:.3f} ms ({48 * pts / f / 1e6:.0f} GB/s), "
          f"accumulating {c:.3f} ms ({56 * pts / c / 1e6:.0f} GB/s)", flush=True)
    del a
    torch.cuda.empty_cache()
