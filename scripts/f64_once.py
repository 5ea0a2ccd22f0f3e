"""A few fp64 gather adjoints of one 3D family (for ncu; developer aid):
    python scripts/f64_once.py [family=wave3d_r4] [n=768]"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1907_02818_b200 import api  # noqa: E402
fam = sys.argv[1] if len(sys.argv) > 1 else "wave3d_r4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 768
a = {nm: torch.randn((n, n, n), dtype=torch.float64, device="cuda")
     for nm in api.array_params(fam, "adjoint")}
for _ in range(3):
    api.adjoint(fam, n, {"D": 0.01 if fam == "wave3d_r4" else 0.1}, a)
torch.cuda.synchronize()
print("ok")
