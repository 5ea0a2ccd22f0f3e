"""A few gather adjoints of one family at a BASELINE size on the bench's own
inputs (for ncu; developer aid):  python scripts/adjoint_once.py <config id>"""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api  # noqa: E402
fam, n, _, _, sc, _ = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "2"]
a = bench.gen_inputs(api, torch, fam, n)
for _ in range(3):
    api.adjoint(fam, n, sc, a)
torch.cuda.synchronize()
print("ok")
