"""One gather and one atomic-scatter adjoint at cfg 4 (for ncu)."""
import sys
sys.path.insert(0, ".")
import torch
import bench
from paper_1907_02818_b200 import api
fam, n = "wave3d_r4", 768
arrays = bench.gen_inputs(api, torch, fam, n)
for _ in range(2):
    api.adjoint(fam, n, {"D": 0.01}, arrays)
    api.scatter_adjoint(fam, n, {"D": 0.01}, arrays)
torch.cuda.synchronize()
print("ok")
