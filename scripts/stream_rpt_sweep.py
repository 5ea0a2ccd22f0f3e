"""Emitted stream form: rows per thread and plane-loop unrolling (developer aid).
python scripts/stream_rpt_sweep.py [n]"""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api, emit_stream, emitter  # noqa: E402
from scripts.quick_time import time_it  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768
for dt in ("f32", "f64"):
    arrays = bench.gen_inputs(api, torch, "wave3d_r4", n, None, dt)
    for tj, rpt, unroll in ((32, 1, False), (16, 1, False), (8, 1, False), (16, 2, False)):
        emit_stream.TJ, emit_stream.RPT, emit_stream.UNROLL = tj, rpt, unroll
        ep = emitter.load_program("wave3d_r4", dt)
        ms = time_it(lambda: ep.adjoint({"n": n}, {"D": 0.01}, arrays, form="stream"),
                     iters=10, warm=2)
        print(f"{dt} tile rows {tj} rows/thread {rpt} unrolled {unroll}: {ms:.3f} ms",
              flush=True)
    del arrays
    torch.cuda.empty_cache()
