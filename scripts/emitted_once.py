"""A few emitted gathers of wave3d_r4 (for ncu; developer aid):
python scripts/emitted_once.py [n] [form=stream|tiled|flat] [dtype=f32]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api, emitter  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
form = sys.argv[2] if len(sys.argv) > 2 else "stream"
dt = sys.argv[3] if len(sys.argv) > 3 else "f32"
arrays = bench.gen_inputs(api, torch, "wave3d_r4", n, None, dt)
ep = emitter.load_program("wave3d_r4", dt)
for _ in range(2):
    ep.adjoint({"n": n}, {"D": 0.01}, arrays, form=form)
torch.cuda.synchronize()
print("ok")
