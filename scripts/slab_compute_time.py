"""Per-rank compute of the z-slab adjoint step on ONE GPU (developer aid):
the launches drivers.adjoint_step issues for an interior rank of an N-way
decomposition (interior planes + two edge bands), halo exchange omitted, vs
the single-GPU step / N.  Estimates the compute side of N-GPU efficiency.
The pipelined form (drivers.HaloPrefetch) is timed with its exchange
emulated by device copies of the same volume on its side stream (the halo
planes in, the owned edge planes out), so HBM / SM contention is included."""
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1907_02818_b200 import api, drivers, slab  # noqa: E402
from scripts.quick_time import time_it as _time_one  # noqa: E402


def time_it(fn, reps=20):
    """ms per call over `reps` back-to-back calls (host launch overhead hidden
    behind queued work, as in a step loop)."""
    return _time_one(lambda: [fn() for _ in range(reps)]) / reps

fam, n = sys.argv[1] if len(sys.argv) > 1 else "wave3d_r4", int(sys.argv[2]) if len(sys.argv) > 2 else 768
R = bench.RADIUS[fam]
sc = {"D": 0.01} if fam == "wave3d_r4" else {"D": 0.1}
full = bench.gen_inputs(api, torch, fam, n)
t1 = time_it(lambda: api.adjoint(fam, n, sc, full))
print(f"{fam} {n}^3 single GPU {t1:.3f} ms")
for N in (2, 4, 8):
    sl = slab.decompose(n, R, N, N // 2)
    loc = bench.gen_inputs(api, torch, fam, n, sl)
    lo_in, hi_in = sl.own0 + R, sl.own1 - R

    def step():
        api.adjoint_slab(fam, n, sc, loc, sl.base, sl.nplanes, lo_in, hi_in)
        api.adjoint_slab(fam, n, sc, loc, sl.base, sl.nplanes, sl.own0, lo_in)
        api.adjoint_slab(fam, n, sc, loc, sl.base, sl.nplanes, hi_in, sl.own1)

    def whole():
        api.adjoint_slab(fam, n, sc, loc, sl.base, sl.nplanes, sl.own0, sl.own1)
    tn = time_it(step)
    tw = time_it(whole)
    top = sl.halo_lo + sl.owned
    nbr = {k: torch.randn((2, R, n, n), device="cuda") for k in ("u_1", "u_b")}

    def exch(ts):  # what NCCL moves: R planes in and out per interior side and field
        for t_, k in zip(ts, ("u_1", "u_b")):
            if sl.halo_lo:
                nbr[k][0].copy_(t_[sl.halo_lo:sl.halo_lo + R])
                t_[:sl.halo_lo].copy_(nbr[k][0])
            if sl.halo_hi:
                nbr[k][1].copy_(t_[top - R:top])
                t_[top:].copy_(nbr[k][1])
    pf = drivers.HaloPrefetch(fam, n, sc, loc, sl, exchange=exch)
    tf = time_it(pf.step)
    pf.close()
    line = (f"  N={N}: rank {N // 2} owns {sl.own1 - sl.own0} planes: overlapped-form compute "
            f"{tn:.3f} ms (eff {t1 / N / tn:.2f}), one launch {tw:.3f} ms (eff {t1 / N / tw:.2f}), "
            f"pipelined (exchange emulated on the side stream) {tf:.3f} ms "
            f"(eff {t1 / N / tf:.2f})")
    if fam == "wave3d_r4":
        # fused peer halo: the neighbours emulated as separate buffers on this GPU
        from paper_1907_02818_b200 import peer
        r = N // 2
        ranks = [q for q in (r - 1, r, r + 1) if 0 <= q < N]
        slabs = [slab.decompose(n, R, N, q) for q in ranks]
        arrs = [bench.gen_inputs(api, torch, fam, n, s2) for s2 in slabs]
        me = ranks.index(r)
        link = peer.emulate(slabs, arrs)[me]
        tp = time_it(lambda: peer.adjoint(n, sc, arrs[me], link))
        line += f", peer {tp:.3f} ms (eff {t1 / N / tp:.2f})"
    print(line)
