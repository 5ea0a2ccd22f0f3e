"""cfg 5 per-rank step on ONE GPU (developer aid): what an interior rank of
an N-way z-slab decomposition does each step -- regenerate u_1 / u_b on its
owned planes (one launch) and the fresh gather over its owned planes (one
launch) -- while its halo exchange is emulated by copy-engine copies of the
same volume on a side stream (R planes of u_1 and u_b in and out per interior
side: what the library's IPC transport pushes), vs the single-GPU step / N.
python scripts/cfg5_rank_time.py [n] [steps] [OPT=V ...]  (options applied to every call)"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1907_02818_b200 import api, drivers, slab  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    api.set_option(k, int(v))
R, fam, sc = 4, "wave3d_r4", {"D": 0.01}


def timed(step, k):
    for t in range(3):
        step(t)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for t in range(k):
        step(t)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / k


a = drivers.alloc(fam, n)
drivers.init_static(fam, a, n, 0)


def one(t):
    drivers.regen_step(a["u_1"], a["u_b"], n, t, 0, R)
    api.adjoint_fresh(fam, n, sc, a)


t1 = timed(one, steps)
print(f"single GPU step {t1:.3f} ms", flush=True)
del a
torch.cuda.empty_cache()
side = torch.cuda.Stream()
for N in (2, 4, 8):
    sl = slab.decompose(n, R, N, N // 2)
    loc = drivers.alloc(fam, n, sl)
    drivers.init_static(fam, loc, n, 0, sl)
    own = slice(sl.own0 - sl.base, sl.own1 - sl.base)
    o = slab.Slab(n, R, sl.rank, sl.world, sl.own0, sl.own1, sl.own0, sl.owned)
    bufs = [torch.empty((R, n, n), device="cuda") for _ in range(8)]

    def rank_step(t):
        drivers.regen_step(loc["u_1"][own], loc["u_b"][own], n, t, 0, R, o)
        ev = torch.cuda.Event()
        ev.record()
        side.wait_event(ev)
        with torch.cuda.stream(side):  # 2 fields x 2 sides x (out + in)
            for k, f in enumerate(("u_1", "u_b")):
                bufs[4 * k].copy_(loc[f][sl.halo_lo:sl.halo_lo + R])
                bufs[4 * k + 1].copy_(loc[f][sl.nplanes - sl.halo_hi - R:sl.nplanes - sl.halo_hi])
                loc[f][:R].copy_(bufs[4 * k + 2])
                loc[f][sl.nplanes - R:].copy_(bufs[4 * k + 3])
        torch.cuda.current_stream().wait_stream(side)
        api.adjoint_slab_fresh(fam, n, sc, loc, sl.base, sl.nplanes, sl.own0, sl.own1)

    tr = timed(rank_step, steps)
    print(f"N={N}: interior rank owns {sl.owned} planes, step {tr:.3f} ms, "
          f"efficiency vs single GPU / N {t1 / N / tr:.2f}", flush=True)
    del loc, bufs
    torch.cuda.empty_cache()
