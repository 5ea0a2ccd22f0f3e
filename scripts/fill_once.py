"""One fill_normal3d at 1024^3 (for ncu; developer aid)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1907_02818_b200 import api  # noqa: E402
a = torch.empty((1024, 1024, 1024), dtype=torch.float32, device="cuda")
for _ in range(3):
    api.fill_normal3d(a, 1024, 4, 0, 1)
torch.cuda.synchronize()
print("ok")
