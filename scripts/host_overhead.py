"""Host-side cost per call of the C-ABI entries and of one pipelined slab step
(developer aid): tiny grids, so the device work is negligible and the wall
time per call is the Python + ctypes + tensor-map encode + launch overhead."""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api, drivers, slab  # noqa: E402

n = 64
a = bench.gen_inputs(api, torch, "wave3d_r4", n)
sc = {"D": 0.01}


def per_call(fn, k=2000):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e6


print(f"api.adjoint (2 launches): {per_call(lambda: api.adjoint('wave3d_r4', n, sc, a)):.1f} us")
sl = slab.decompose(n, 4, 4, 1)
loc = bench.gen_inputs(api, torch, "wave3d_r4", n, sl)
print(f"api.adjoint_slab: "
      f"{per_call(lambda: api.adjoint_slab('wave3d_r4', n, sc, loc, sl.base, sl.nplanes, sl.own0, sl.own1)):.1f} us")
top = sl.halo_lo + sl.owned


def exch(ts):
    for t_ in ts:
        t_[:sl.halo_lo].copy_(t_[sl.halo_lo:sl.halo_lo + 4])
        t_[top:].copy_(t_[top - 4:top])


pf = drivers.HaloPrefetch("wave3d_r4", n, sc, loc, sl, exchange=exch)
print(f"HaloPrefetch.step (emulated exchange: 4 copies): {per_call(pf.step):.1f} us")
pf.close()
