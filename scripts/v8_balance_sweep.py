"""Split point of the balanced v8 interior launch (V8_BALANCE=m forces it):
python scripts/v8_balance_sweep.py n m1 m2 ..."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers  # noqa: E402

n = int(sys.argv[1])
ms = [int(x) for x in sys.argv[2:]]
a = drivers.alloc("wave3d_r4", n)
drivers.init_static("wave3d_r4", a, n, 0)
drivers.regen_step(a["u_1"], a["u_b"], n, 0, 0, 4)
res = {m: [] for m in ms}
for rnd in range(7):
    for m in (ms if rnd % 2 == 0 else ms[::-1]):
        with api.options(V8_BALANCE=m):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            for i in range(5):
                ev[i].record()
                api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a)
            ev[5].record()
            torch.cuda.synchronize()
        if rnd:
            res[m] += [ev[i].elapsed_time(ev[i + 1]) for i in range(5)]
        time.sleep(0.3)
for m in ms:
    print(f"n={n} V8_BALANCE={m}: {statistics.median(res[m]):.3f} ms", flush=True)
