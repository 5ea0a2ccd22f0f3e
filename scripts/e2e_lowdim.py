"""e2e (host-buffer plan) of cfg 1 / cfg 3 vs chunk count (developer aid):
    python scripts/e2e_lowdim.py"""
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")
if len(sys.argv) > 1:
    import bench
    from paper_1907_02818_b200 import api
    cid = sys.argv[1]
    fam, n, dt, _, sc, _ = bench.CONFIGS[cid]
    d = bench.DIMS[fam]
    tdt = torch.float64 if dt == "f64" else torch.float32
    host = {nm: torch.randn((n,) * d, dtype=tdt).pin_memory()
            for nm in api.array_params(fam, "adjoint", dt)}
    plan = api.Plan(fam, n, dt)
    plan.run_adjoint_host(sc, host)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        plan.run_adjoint_host(sc, host)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"cfg{cid} chunks={os.environ.get('SGB_PLAN_CHUNKS', 'default')} e2e {ms:.2f} ms "
          f"{n ** d / ms / 1e6:.2f} GPts/s")
    sys.exit(0)
for cid in ("1", "3"):
    for c in ("1", "8", "32", "64"):
        subprocess.run([sys.executable, __file__, cid], env=dict(os.environ, SGB_PLAN_CHUNKS=c),
                       check=True)
