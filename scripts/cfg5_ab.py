"""A/B of run-time options on cfg 5's step (regenerate u_1 / u_b, fused fresh
gather) at n^3, sustained: variants interleaved round-robin, `steps` back-to-
back steps per round, CUDA events around the gather and the whole step
(AB_PAUSE=seconds between runs: burst clocks instead of the power-capped state).
python scripts/cfg5_ab.py n steps rounds "" "V7_UNIFIED=1" "ICHUNKS=2,ICHUNKS_F=4" ..."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402

n, steps, rounds = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
variants = sys.argv[4:] or [""]
a = drivers.alloc("wave3d_r4", n)
drivers.init_static("wave3d_r4", a, n, 0)


def parse(v):
    out = {}
    for kv in filter(None, v.split(",")):
        k, x = kv.split("=")
        out[k] = int(x)
    return out


res = {v: ([], []) for v in variants}
for r in range(rounds + 1):
    for v in (variants if r % 2 == 0 else variants[::-1]):  # no position bias
        with api.options(**parse(v)):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
                   torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for t in range(steps):
                ev[t][0].record()
                drivers.regen_step(a["u_1"], a["u_b"], n, t, 0, 4)
                ev[t][1].record()
                api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a)
                ev[t][2].record()
            torch.cuda.synchronize()
        if os.environ.get("AB_PAUSE"):  # burst mode: let the board cool between runs
            time.sleep(float(os.environ["AB_PAUSE"]))
        if r == 0:
            continue  # warm-up round
        res[v][0].extend(e1.elapsed_time(e2) for _, e1, e2 in ev)
        res[v][1].extend(e0.elapsed_time(e2) for e0, _, e2 in ev)
for v, (g, s) in res.items():
    print(f"{v or 'default':40s} gather median {statistics.median(g):.3f} ms  "
          f"step median {statistics.median(s):.3f} ms  (n={len(g)})")
