"""Timing of the emitted generic gather at cfg 4 (developer aid): the tiled
form (shared-memory rings of the factored Q field and the u_1 planes) and the
one-thread-per-point form, fp32 and fp64, beside the hand-tuned kernel.
python scripts/emitted_time.py [n]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api, emitter  # noqa: E402
from scripts.quick_time import time_it  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
for dt in ("f32", "f64"):
    arrays = bench.gen_inputs(api, torch, "wave3d_r4", n, None, dt)
    ep = emitter.load_program("wave3d_r4", dt)
    hand = time_it(lambda: api.adjoint("wave3d_r4", n, {"D": 0.01}, arrays), iters=10, warm=2)
    out = [f"{dt} {n}^3: hand-tuned {hand:.3f} ms"]
    for form in ("stream", "tiled", "flat"):
        ms = time_it(lambda: ep.adjoint({"n": n}, {"D": 0.01}, arrays, form=form), iters=10,
                     warm=2)
        out.append(f"emitted {form} {ms:.3f} ms ({ms / hand:.2f}x)")
    print(", ".join(out), flush=True)
    del arrays
    torch.cuda.empty_cache()
