"""v8 interior with the balanced last wave (V8_BALANCE=1, default) vs the plain
launch: bitwise equality and timing (alternating order, burst pauses).
python scripts/v8_balance_check.py n1 n2 ..."""
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
    base = a["c_b"].clone()
    outs = {}
    for v in (0, 1):
        a["c_b"].copy_(base)
        a["u_1_b"].fill_(float("nan"))
        with api.options(V8_BALANCE=v):
            api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a)
        torch.cuda.synchronize()
        outs[v] = {k: a[k].clone() for k in ("c_b", "u_1_b")}
    for k in ("c_b", "u_1_b"):
        print(f"n={n} {k}: bitwise equal "
              f"{torch.equal(outs[0][k].view(torch.int32), outs[1][k].view(torch.int32))}",
              flush=True)
    res = {0: [], 1: []}
    for rnd in range(9):
        for v in ((0, 1) if rnd % 2 == 0 else (1, 0)):
            with api.options(V8_BALANCE=v):
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
                for i in range(5):
                    ev[i].record()
                    api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a)
                ev[5].record()
                torch.cuda.synchronize()
            if rnd:
                res[v] += [ev[i].elapsed_time(ev[i + 1]) for i in range(5)]
            time.sleep(0.5)
    m0, m1 = statistics.median(res[0]), statistics.median(res[1])
    print(f"n={n} fresh gather: plain {m0:.3f} ms, balanced {m1:.3f} ms ({m1 / m0:.3f})", flush=True)
    del a, base, outs
    torch.cuda.empty_cache()
