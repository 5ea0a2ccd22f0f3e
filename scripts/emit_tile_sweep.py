import sys
import torch
sys.path.insert(0, ".")
import bench
from paper_1907_02818_b200 import api, emitter
from scripts.quick_time import time_it
n = 768
for dt in ("f32", "f64"):
    arrays = bench.gen_inputs(api, torch, "wave3d_r4", n, None, dt)
    hand = time_it(lambda: api.adjoint("wave3d_r4", n, {"D": 0.01}, arrays), iters=10, warm=2)
    for ty in (8, 16, 24, 32):
        emitter.EmittedProblem.TILE_Y = ty
        ep = emitter.load_program("wave3d_r4", dt)
        if ep.tiled_layout() is None:
            print(dt, ty, "no layout"); continue
        ms = time_it(lambda: ep.adjoint({"n": n}, {"D": 0.01}, arrays, form="tiled"), iters=10, warm=2)
        print(f"{dt} TILE_Y={ty} smem={ep.tiled_layout()['smem']} tiled {ms:.3f} ms ({ms/hand:.2f}x hand {hand:.3f})", flush=True)
    del arrays; torch.cuda.empty_cache()
