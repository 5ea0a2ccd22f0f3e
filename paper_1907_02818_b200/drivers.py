"""Multi-step reverse drivers for the BASELINE configs (host orchestration).

The hot path is the C-ABI gather adjoint; these drivers are the plumbing a
solver's time loop provides around it (the paper's ``printfunction`` caller,
PAPER.md:352-354), following SURVEY Appendix B:

* cfg 5 (``run_independent``): wave3d_r4, N reverse steps; each step
  regenerates the forward state u_1 = u^t and the seed u_b from (seed, t),
  exchanges their radius-4 halos (z-slab), zeroes u_1_b and runs the gather
  adjoint, accumulating c_b over all steps (the time-integrated c gradient).
* cfg 2 (``run_carried``): wave3d_c, N carried reverse steps; step t uses the
  seed u_b = u-bar^{t+1}, accumulates u_1_b = u-bar^t, u_2_b = u-bar^{t-1} and
  c_b, then rotates seed <- u_1_b, u_1_b <- u_2_b, u_2_b <- 0; u_1 = u^t is
  regenerated from (seed, t).
* ``adjoint_step``: one z-slab step with the halo exchange overlapped with the
  interior planes (whose stencils never touch a halo), then the edge planes.

Generators are counter-based in the global index, so any decomposition sees
the single-GPU inputs (tests regenerate them with the same calls).
"""
from __future__ import annotations

import torch

from . import api
from . import slab as slabmod

R_OF = {"wave3d_r4": 4, "wave3d_c": 1, "wave3d_c2": 1}


def _planes(sl, n):
    return (sl.base, sl.nplanes) if sl is not None else (0, n)


def regen_state(u_1, n, t, seed, radius, sl=None):
    """u^t ~ N(0,1) with a zero `radius`-point halo, from (seed, step t)."""
    base, npl = _planes(sl, n)
    api.fill_normal3d(u_1, n, radius, seed, 1000 + 2 * t, base, npl)


def regen_seed(u_b, n, t, seed, sl=None):
    base, npl = _planes(sl, n)
    api.fill_normal3d(u_b, n, 0, seed, 1001 + 2 * t, base, npl)


def adjoint_step(family, n, scalars, arrays, sl=None, exchange=("u_1", "u_b"), overlap=True):
    """One gather-adjoint step; with a slab, halos of `exchange` are refreshed
    first -- overlapped with the interior planes when `overlap`."""
    if sl is None:
        api.adjoint(family, n, scalars, arrays)
        return 1
    R = sl.radius
    lo_in, hi_in = sl.own0 + (R if sl.rank > 0 else 0), sl.own1 - (R if sl.rank < sl.world - 1 else 0)
    fields = [arrays[k] for k in exchange]
    if not overlap or hi_in <= lo_in or sl.world == 1:
        slabmod.exchange_halos(sl, fields)
        api.adjoint_slab(family, n, scalars, arrays, sl.base, sl.nplanes, sl.own0, sl.own1)
        return 1
    import torch.distributed as dist
    ops = slabmod.halo_ops(sl, fields)
    reqs = dist.batch_isend_irecv(ops)
    # interior planes: their stencils only read owned planes
    api.adjoint_slab(family, n, scalars, arrays, sl.base, sl.nplanes, lo_in, hi_in)
    for r in reqs:
        r.wait()
    launches = 1
    if lo_in > sl.own0:
        api.adjoint_slab(family, n, scalars, arrays, sl.base, sl.nplanes, sl.own0, lo_in)
        launches += 1
    if hi_in < sl.own1:
        api.adjoint_slab(family, n, scalars, arrays, sl.base, sl.nplanes, hi_in, sl.own1)
        launches += 1
    return launches


def alloc(family, n, sl=None, dtype=torch.float32):
    shape = (sl.nplanes, n, n) if sl is not None else (n, n, n)
    return {nm: torch.zeros(shape, dtype=dtype, device="cuda")
            for nm in api.array_params(family, "adjoint")}


def init_static(family, arrays, n, seed=0, sl=None):
    """c: layered U[1.5,4.5] on 8 z-layers (cfg 4/5) or U[1.5,4.5] (cfg 2)."""
    base, npl = _planes(sl, n)
    if family == "wave3d_r4":
        api.fill_layered(arrays["c"], n, 8, 1.5, 4.5, seed, base, npl)
    else:
        api.fill_random(arrays["c"], base * n * n, seed, 0, "uniform", 1.5, 3.0)


def run_independent(n, steps, seed=0, D=0.01, sl=None, arrays=None, overlap=True):
    """cfg 5: independent reverse steps of wave3d_r4, c_b accumulated."""
    fam = "wave3d_r4"
    if arrays is None:
        arrays = alloc(fam, n, sl)
        init_static(fam, arrays, n, seed, sl)
    for t in range(steps):
        regen_state(arrays["u_1"], n, t, seed, 4, sl)
        regen_seed(arrays["u_b"], n, t, seed, sl)
        arrays["u_1_b"].zero_()
        adjoint_step(fam, n, {"D": D}, arrays, sl, overlap=overlap)
    return arrays


def run_carried(n, steps, seed=0, D=0.1, family="wave3d_c", arrays=None):
    """cfg 2: carried reverse steps of the 7-point wave (single GPU)."""
    if arrays is None:
        arrays = alloc(family, n)
        init_static(family, arrays, n, seed)
        regen_seed(arrays["u_b"], n, steps, seed)  # u-bar^{T+1}
    for t in reversed(range(steps)):
        regen_state(arrays["u_1"], n, t, seed, 1)
        api.adjoint(family, n, {"D": D}, arrays)
        # rotate: seed <- u_1_b, u_1_b <- u_2_b, u_2_b <- 0
        arrays["u_b"], arrays["u_1_b"], arrays["u_2_b"] = (arrays["u_1_b"], arrays["u_2_b"],
                                                           arrays["u_b"])
        arrays["u_2_b"].zero_()
    return arrays
