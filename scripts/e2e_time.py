"""Scratch timing of the host-buffer entry (developer aid, not the bench):
raw pinned H2D / D2H bandwidth and sgb_plan_run_adjoint_host per chunk count."""
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 768


def ev_time(fn, k=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(k):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / k


if len(sys.argv) > 2:  # child: one chunk setting
    names = api.array_params("wave3d_r4", "adjoint")
    host = {nm: torch.randn((n, n, n), dtype=torch.float32).pin_memory() for nm in names}
    plan = api.Plan("wave3d_r4", n, "f32")
    ms = ev_time(lambda: plan.run_adjoint_host({"D": 0.01}, host))
    print(f"chunks={os.environ.get('SGB_PLAN_CHUNKS')} e2e {ms:.1f} ms "
          f"{n**3 / ms / 1e6:.2f} GPts/s")
    sys.exit(0)

h = torch.empty(n ** 3, dtype=torch.float32).pin_memory()
d = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
gb = h.numel() * 4 / 1e9
print(f"H2D {gb / ev_time(lambda: d.copy_(h, non_blocking=True)) * 1e3:.1f} GB/s, "
      f"D2H {gb / ev_time(lambda: h.copy_(d, non_blocking=True)) * 1e3:.1f} GB/s")
# the plan's copy pattern without the kernel: H2D of all five arrays, and the
# same H2D with D2H of two arrays concurrently on a second stream (PCIe is
# full duplex; what the concurrent direction costs the H2D side is the floor)
hs = [torch.empty(n ** 3, dtype=torch.float32).pin_memory() for _ in range(5)]
ds = [torch.empty(n ** 3, dtype=torch.float32, device="cuda") for _ in range(5)]
s2 = torch.cuda.Stream()


def h2d_all():
    for a, b in zip(ds, hs):
        a.copy_(b, non_blocking=True)


def both():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        for k in (1, 3):
            hs[k].copy_(ds[k], non_blocking=True)
    h2d_all()
    torch.cuda.current_stream().wait_stream(s2)


t1, t2 = ev_time(h2d_all), ev_time(both)
print(f"H2D of 5 arrays {t1:.1f} ms ({5 * gb / t1 * 1e3:.1f} GB/s); with D2H of 2 arrays "
      f"concurrently {t2:.1f} ms ({5 * gb / t2 * 1e3:.1f} GB/s H2D)")
del h, d, hs, ds
for c in (8, 16, 32, 64):
    subprocess.run([sys.executable, __file__, str(n), "child"],
                   env=dict(os.environ, SGB_PLAN_CHUNKS=str(c)), check=True)
