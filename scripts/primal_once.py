"""One radius-4 primal at 768^3 fp32 (for ncu; developer aid)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1907_02818_b200 import api  # noqa: E402
n = 768
a = {nm: torch.randn((n, n, n), device="cuda") for nm in api.array_params("wave3d_r4", "primal")}
for _ in range(3):
    api.primal("wave3d_r4", n, {"D": 0.01}, a)
torch.cuda.synchronize()
print("ok")
