"""Scratch timing of the emitted generic gather at cfg 4 (developer aid)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api, emitter  # noqa: E402
from scripts.quick_time import time_it  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
arrays = bench.gen_inputs(api, torch, "wave3d_r4", n)
ep = emitter.load_program("wave3d_r4", "f32")
ms = time_it(lambda: ep.adjoint({"n": n}, {"D": 0.01}, arrays), iters=10, warm=2)
print(f"emitted fused gather {n}^3: {ms:.3f} ms")
