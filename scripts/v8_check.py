"""Experimental v8 interior kernel vs v7 (developer aid): result difference
(fp32 rounding only) and timing, alternating order, burst pauses.
python scripts/v8_check.py n1 n2 ..."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402

for n in (int(x) for x in sys.argv[1:]):
    a = drivers.alloc("wave3d_r4", n)
    drivers.init_static("wave3d_r4", a, n, 0)
    drivers.regen_step(a["u_1"], a["u_b"], n, 0, 0, 4)
    api.fill_random(a["c_b"], 0, 3, 1, "normal", 0.0, 1.0)
    api.fill_random(a["u_1_b"], 0, 3, 2, "normal", 0.0, 1.0)
    base = {k: a[k].clone() for k in ("c_b", "u_1_b")}
    for kind, call in (("acc", api.adjoint), ("fresh", api.adjoint_fresh)):
        outs = {}
        for v8 in (0, 1):
            for k in base:
                a[k].copy_(base[k])
            with api.options(V8_INTERIOR=v8):
                call("wave3d_r4", n, {"D": 0.01}, a)
            torch.cuda.synchronize()
            outs[v8] = {k: a[k].double().clone() for k in base}
        for k in base:
            d = (outs[1][k] - outs[0][k]).abs()
            rel = float((d / (1 + outs[0][k].abs())).max())
            same = torch.equal(outs[1][k], outs[0][k])
            print(f"n={n} {kind} {k}: max |v8-v7|/(1+|v7|) = {rel:.2e}, bitwise equal {same}",
                  flush=True)
        res = {0: [], 1: []}
        for rnd in range(7):
            for v8 in ((0, 1) if rnd % 2 == 0 else (1, 0)):
                with api.options(V8_INTERIOR=v8):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
                    for i in range(10):
                        ev[i].record()
                        call("wave3d_r4", n, {"D": 0.01}, a)
                    ev[10].record()
                    torch.cuda.synchronize()
                if rnd:
                    res[v8] += [ev[i].elapsed_time(ev[i + 1]) for i in range(10)]
                time.sleep(0.5)
        m0, m1 = statistics.median(res[0]), statistics.median(res[1])
        print(f"n={n} {kind}: v7 {m0:.3f} ms, v8 interior {m1:.3f} ms ({m1 / m0:.3f})",
              flush=True)
    del a, base
    torch.cuda.empty_cache()
