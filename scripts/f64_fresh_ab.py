"""fp64 fresh radius-4 gather: time + output digest of the loaded library
(SGB_LIB_PATH selects another build for an A/B):
python scripts/f64_fresh_ab.py n1 n2 ..."""
import hashlib
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
    api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a)
    torch.cuda.synchronize()
    h = hashlib.sha1()
    for k in ("c_b", "u_1_b"):
        h.update(a[k].cpu().numpy().tobytes())
    ts = []
    for rnd in range(6):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        for i in range(5):
            ev[i].record()
            api.adjoint_fresh("wave3d_r4", n, {"D": 0.01}, a)
        ev[5].record()
        torch.cuda.synchronize()
        if rnd:
            ts += [ev[i].elapsed_time(ev[i + 1]) for i in range(5)]
        time.sleep(0.5)
    print(f"n={n} fresh fp64: {statistics.median(ts):.3f} ms  digest {h.hexdigest()[:16]}", flush=True)
    del a
    torch.cuda.empty_cache()
