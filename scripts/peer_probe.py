"""Developer aid: the fused-halo (peer) launch vs the plain slab launch on one
GPU (neighbours emulated as separate buffers)."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api, peer, slab  # noqa: E402
from scripts.quick_time import time_it as _one  # noqa: E402


def time_it(fn, reps=20):
    return _one(lambda: [fn() for _ in range(reps)]) / reps


n, N = 768, 2
sc = {"D": 0.01}
slabs = [slab.decompose(n, 4, N, q) for q in range(N)]
arrs = [bench.gen_inputs(api, torch, "wave3d_r4", n, s) for s in slabs]
links = peer.emulate(slabs, arrs)
sl, a = slabs[1], arrs[1]
t_whole = time_it(lambda: api.adjoint_slab("wave3d_r4", n, sc, a, sl.base, sl.nplanes,
                                           sl.own0, sl.own1))
t_peer = time_it(lambda: peer.adjoint(n, sc, a, links[1]))
print(f"slab call incl. halos {t_whole:.3f} ms | peer (halo planes from the neighbour's "
      f"arrays) {t_peer:.3f} ms")
