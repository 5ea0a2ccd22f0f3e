"""L2-prefetch distance of the radius-4 gather vs grid size (developer aid):
python scripts/pf_sweep.py [--acc] n1 n2 ...  (fresh gather, or the accumulating
one with --acc; burst: 0.5 s pause per run, variant order alternating)"""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402

acc = "--acc" in sys.argv
call = api.adjoint if acc else api.adjoint_fresh
for n in (int(x) for x in sys.argv[1:] if not x.startswith("--")):
    a = drivers.alloc("wave3d_r4", n)
    drivers.init_static("wave3d_r4", a, n, 0)
    drivers.regen_step(a["u_1"], a["u_b"], n, 0, 0, 4)
    res = {0: [], 1: [], 2: []}
    for rnd in range(6):
        for pf in (list(res) if rnd % 2 == 0 else list(res)[::-1]):
            with api.options(V7_PREFETCH=pf):
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
                for i in range(10):
                    ev[i].record()
                    call("wave3d_r4", n, {"D": 0.01}, a)
                ev[10].record()
                torch.cuda.synchronize()
            if rnd:
                res[pf] += [ev[i].elapsed_time(ev[i + 1]) for i in range(10)]
            time.sleep(0.5)
    base = statistics.median(res[0])
    print(f"n={n}: " + ", ".join(f"PF={pf} {statistics.median(v):.3f} ms "
                                 f"({statistics.median(v) / base:.3f})" for pf, v in res.items()),
          flush=True)
    del a
    torch.cuda.empty_cache()
