"""fp64 radius-4 gather: the v8 form (F64_V8=1, default) vs the 2-row form
(F64_V8=0): bitwise equality and timing, alternating order, burst pauses.
python scripts/f64v8_check.py n1 n2 ..."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api  # noqa: E402

for n in (int(x) for x in sys.argv[1:]):
    g = torch.Generator(device="cuda").manual_seed(n)
    a = {k: torch.randn((n, n, n), generator=g, device="cuda", dtype=torch.float64)
         for k in ("c", "c_b", "u_1", "u_1_b", "u_b")}
    base = {k: a[k].clone() for k in ("c_b", "u_1_b")}
    for kind, call in (("acc", api.adjoint), ("fresh", api.adjoint_fresh)):
        outs = {}
        for v in (0, 1):
            for k in base:
                a[k].copy_(base[k])
            with api.options(F64_V8=v):
                call("wave3d_r4", n, {"D": 0.01}, a)
            torch.cuda.synchronize()
            outs[v] = {k: a[k].clone() for k in base}
        for k in base:
            print(f"n={n} {kind} {k}: bitwise equal "
                  f"{torch.equal(outs[0][k].view(torch.int64), outs[1][k].view(torch.int64))}",
                  flush=True)
        res = {0: [], 1: []}
        for rnd in range(7):
            for v in ((0, 1) if rnd % 2 == 0 else (1, 0)):
                with api.options(F64_V8=v):
                    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
                    for i in range(5):
                        ev[i].record()
                        call("wave3d_r4", n, {"D": 0.01}, a)
                    ev[5].record()
                    torch.cuda.synchronize()
                if rnd:
                    res[v] += [ev[i].elapsed_time(ev[i + 1]) for i in range(5)]
                time.sleep(0.5)
        m0, m1 = statistics.median(res[0]), statistics.median(res[1])
        print(f"n={n} {kind}: 2-row {m0:.3f} ms, v8 {m1:.3f} ms ({m1 / m0:.3f})", flush=True)
    del a, base
    torch.cuda.empty_cache()
