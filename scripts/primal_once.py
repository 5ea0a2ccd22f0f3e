"""A few primal calls of one family (for ncu; developer aid):
    python scripts/primal_once.py [family=wave3d_r4] [n=768]"""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api  # noqa: E402
fam = sys.argv[1] if len(sys.argv) > 1 else "wave3d_r4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 768
d = bench.DIMS[fam]
dt = torch.float32 if fam.startswith("wave3d") else torch.float64
a = {nm: torch.randn((n,) * d, device="cuda", dtype=dt) for nm in api.array_params(fam, "primal")}
sc = {"D": 0.01 if fam == "wave3d_r4" else 0.1, "C": 0.2}
if fam == "burgers2d":
    sc["D"] = 0.002
for _ in range(3):
    api.primal(fam, n, sc, a)
torch.cuda.synchronize()
print("ok")
