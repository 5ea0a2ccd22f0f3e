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


def regen_step(u_1, u_b, n, t, seed, radius, sl=None):
    """regen_state + regen_seed of step t in one pass (bitwise the same values)."""
    base, npl = _planes(sl, n)
    api.fill_normal3d_pair(u_1, radius, 1000 + 2 * t, u_b, 0, 1001 + 2 * t, n, seed, base, npl)


def adjoint_step(family, n, scalars, arrays, sl=None, exchange=("u_1", "u_b"), overlap=True,
                 link=None, fresh=False):
    """One gather-adjoint step; with a slab, halos of `exchange` are refreshed
    first -- overlapped with the interior planes when `overlap` -- or, with a
    peer `link` (peer.try_connect), read by the kernel straight from the
    neighbours' arrays after a stream-ordered cross-rank sync."""
    if fresh and link is not None:
        raise ValueError("fresh u_1_b is not available on the peer-halo path")
    if sl is None:
        (api.adjoint_fresh if fresh else api.adjoint)(family, n, scalars, arrays)
        return 1
    slab_call = api.adjoint_slab_fresh if fresh else api.adjoint_slab
    if link is not None:
        from . import peer
        peer.step_sync()
        peer.adjoint(n, scalars, arrays, link)
        return 1
    R = sl.radius
    lo_in, hi_in = sl.own0 + (R if sl.rank > 0 else 0), sl.own1 - (R if sl.rank < sl.world - 1 else 0)
    fields = [arrays[k] for k in exchange]
    if not overlap or hi_in <= lo_in or sl.world == 1:
        slabmod.exchange_halos(sl, fields)
        slab_call(family, n, scalars, arrays, sl.base, sl.nplanes, sl.own0, sl.own1)
        return 1
    import torch.distributed as dist
    ops = slabmod.halo_ops(sl, fields)
    reqs = dist.batch_isend_irecv(ops)
    # interior planes: their stencils only read owned planes
    slab_call(family, n, scalars, arrays, sl.base, sl.nplanes, lo_in, hi_in)
    for r in reqs:
        r.wait()
    launches = 1
    if lo_in > sl.own0:
        slab_call(family, n, scalars, arrays, sl.base, sl.nplanes, sl.own0, lo_in)
        launches += 1
    if hi_in < sl.own1:
        slab_call(family, n, scalars, arrays, sl.base, sl.nplanes, hi_in, sl.own1)
        launches += 1
    return launches


class HaloPrefetch:
    """Cross-step pipelined halo exchange for z-slab steps whose
    inputs do not depend on the previous step's outputs -- cfg 4 (the same
    forward state and seed every step) and cfg 5 (both regenerated from
    (seed, step)).  The exchanged fields (u_1, u_b) get two buffer sets: while
    the gather adjoint of step t reads set t % 2 in ONE launch over the owned
    planes (halos already in place), a high-priority side stream regenerates
    step t+1's owned planes into the other set (cfg 5) and exchanges that
    set's halo planes with the neighbours (NCCL over NVLink), so the exchange
    -- and the regeneration -- run behind the compute instead of before it.
    Step t still consumes exactly the planes the exchange-then-compute path
    gives it, so the outputs are bitwise identical (tests/test_drivers_gpu.py).

    regen(fields, t): writes step t's owned planes of the exchanged fields
    (None: inputs static); exchange(tensors): refreshes their halo planes
    (default: slab.exchange_halos, one batched NCCL isend/irecv round).
    Call step(t) for t = 0, 1, 2, ... on the compute stream; close() drains
    the side stream."""

    def __init__(self, family, n, scalars, arrays, sl, fields=("u_1", "u_b"), regen=None,
                 exchange=None, fresh=False, compute=None):
        self.family, self.n, self.scalars, self.arrays, self.sl = family, n, scalars, arrays, sl
        self.fresh = fresh  # u_1_b = this step's adjoint alone (cfg 5)
        self.fields = tuple(fields)
        self.regen = regen
        self.exchange = exchange or (lambda ts: slabmod.exchange_halos(sl, ts))
        # compute(inputs, t): the step's kernel (default: the slab gather);
        # CPU tensors (the gloo tests of the exchange schedule) run it and
        # the preparation in program order, without streams or events
        self.compute = compute
        # both sets are private copies (initialised from `arrays`), so the
        # side stream never writes a tensor the caller may still use
        self.sets = [{f: arrays[f].clone() for f in self.fields} for _ in range(2)]
        self.cuda = arrays[self.fields[0]].is_cuda
        if self.cuda:
            self.side = torch.cuda.Stream(priority=-1)
            self.ready = [torch.cuda.Event(), torch.cuda.Event()]
            self.free = [torch.cuda.Event(), torch.cuda.Event()]
            self.side.wait_stream(torch.cuda.current_stream())  # arrays initialised
        self._t = 0
        self._prepare(0)
        self._prepare(1)

    def _prepare(self, t):
        s = t % 2
        if not self.cuda:
            if self.regen is not None:
                self.regen(self.sets[s], t)
            self.exchange([self.sets[s][f] for f in self.fields])
            return
        with torch.cuda.stream(self.side):
            if t >= 2:  # step t-2 finished reading this set
                self.side.wait_event(self.free[s])
            if self.regen is not None:
                self.regen(self.sets[s], t)
            self.exchange([self.sets[s][f] for f in self.fields])
            self.ready[s].record(self.side)

    def inputs(self, t):
        """The arrays step t reads (the static ones + set t % 2)."""
        a = dict(self.arrays)
        a.update(self.sets[t % 2])
        return a

    def step(self, t=None):
        """Step t's gather adjoint (one launch over the owned planes) on the
        current stream; enqueues step t+2's input preparation behind it."""
        t = self._t if t is None else t
        if t != self._t:
            raise ValueError(f"HaloPrefetch steps run in order: expected {self._t}, got {t}")
        s = t % 2
        sl = self.sl
        if self.cuda:
            cur = torch.cuda.current_stream()
            cur.wait_event(self.ready[s])
        if self.compute is not None:
            self.compute(self.inputs(t), t)
        else:
            call = api.adjoint_slab_fresh if self.fresh else api.adjoint_slab
            call(self.family, self.n, self.scalars, self.inputs(t), sl.base, sl.nplanes,
                 sl.own0, sl.own1)
        if self.cuda:
            self.free[s].record(cur)
        self._t = t + 1
        self._prepare(t + 2)
        return 1

    def close(self):
        if self.cuda:
            torch.cuda.current_stream().wait_stream(self.side)
            self.side.synchronize()


class PlanPrefetch:
    """HaloPrefetch on the library's own z-slab plan (slab.SlabPlan; the
    exchange is the plan's NCCL or CUDA-IPC transport, sgb_slab_halo_start):
    the u_1 / u_b inputs of step t live in buffer set t % 2 (both sets bound
    to the plan); a high-priority side stream regenerates step t+1's owned
    planes and starts that set's halo exchange while step t's single launch
    over the owned planes reads the other set.  Same inputs per step as the
    exchange-then-compute path, so the outputs are bitwise equal (tested).

    plan: a connected SlabPlan whose set 0 / 1 are `sets[0]` / `sets[1]`
    (dicts with "u_1", "u_b"); regen(fields, t) writes step t's OWNED planes
    (None: static inputs, the halos are still refreshed every step)."""

    def __init__(self, plan, scalars, sets, regen=None, fresh=False):
        self.plan, self.scalars, self.sets = plan, scalars, sets
        self.regen, self.fresh = regen, fresh
        self.side = torch.cuda.Stream(priority=-1)
        self.free = [torch.cuda.Event(), torch.cuda.Event()]
        self.side.wait_stream(torch.cuda.current_stream())
        self._t = 0
        self._prepare(0)
        self._prepare(1)

    def _prepare(self, t):
        s = t % 2
        with torch.cuda.stream(self.side):
            if t >= 2:  # step t-2 finished reading this set on this rank
                self.side.wait_event(self.free[s])
            if self.regen is not None:
                self.regen(self.sets[s], t)
            self.plan.halo_start(("u_1", "u_b"), s, stream=self.side)

    def step(self, t=None):
        t = self._t if t is None else t
        if t != self._t:
            raise ValueError(f"PlanPrefetch steps run in order: expected {self._t}, got {t}")
        s = t % 2
        cur = torch.cuda.current_stream()
        self.plan.step(self.scalars, set_=s, fresh=self.fresh, exchanged=True, stream=cur)
        self.free[s].record(cur)
        self._t = t + 1
        self._prepare(t + 2)
        return 1

    def close(self):
        torch.cuda.current_stream().wait_stream(self.side)
        self.side.synchronize()


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


def run_independent(n, steps, seed=0, D=0.01, sl=None, arrays=None, overlap=True, fresh=True):
    """cfg 5: independent reverse steps of wave3d_r4, c_b accumulated."""
    fam = "wave3d_r4"
    if arrays is None:
        arrays = alloc(fam, n, sl)
        init_static(fam, arrays, n, seed, sl)
    for t in range(steps):
        regen_step(arrays["u_1"], arrays["u_b"], n, t, seed, 4, sl)
        if fresh:  # u_1_b = this step's adjoint: zeroing fused into the gather
            adjoint_step(fam, n, {"D": D}, arrays, sl, overlap=overlap, fresh=True)
        else:
            arrays["u_1_b"].zero_()
            adjoint_step(fam, n, {"D": D}, arrays, sl, overlap=overlap)
    return arrays


def run_carried(n, steps, seed=0, D=0.1, family="wave3d_c", arrays=None):
    """cfg 2: carried reverse steps of the 7-point wave (single GPU).  On
    return u_b = u-bar^0 (the last step's u_1_b), u_1_b = u-bar^{-1} (its u_2
    partial) and u_2_b = 0, whichever path ran.  Caller-supplied `arrays`
    keep their u_1_b / u_2_b / c_b contents as the initial accumulators."""
    caller = arrays is not None
    if arrays is None:
        arrays = alloc(family, n)
        init_static(family, arrays, n, seed)
        regen_seed(arrays["u_b"], n, steps, seed)  # u-bar^{T+1}
    fused = arrays["u_1"].dtype == torch.float32
    for k, t in enumerate(reversed(range(steps))):
        regen_state(arrays["u_1"], n, t, seed, 1)
        # u_2_b written as this step's partial (the zeroing below, fused); a
        # caller's first step accumulates into whatever u_2_b it passed
        if fused and not (caller and k == 0):
            api.adjoint_fresh_u2(family, n, {"D": D}, arrays)
        else:
            api.adjoint(family, n, {"D": D}, arrays)
        # rotate: seed <- u_1_b, u_1_b <- u_2_b, u_2_b <- 0 (on the fused path
        # the zeroing is folded into the next step's gather, and done once
        # after the sweep)
        arrays["u_b"], arrays["u_1_b"], arrays["u_2_b"] = (arrays["u_1_b"], arrays["u_2_b"],
                                                           arrays["u_b"])
        if not fused or k == steps - 1:
            arrays["u_2_b"].zero_()
    return arrays


# ---------------------------------------------------------------------------
# the adjoint of a whole wave3d_r4 time loop with REAL
# forward recomputation from uniform checkpoints (the reference's scope ends
# at one loop nest; a solver's time loop is what surrounds it).
#
#   forward   u^{t+1} = 2 u^t - u^{t-1} + c^2 D Lap25(u^t)   (primal kernel)
#   loss      J = <w, u^T>
#   reverse   for t = T-1 .. 1:
#               c_b += dF/dc^T u-bar^{t+1};  u-bar^t += dF/du^t^T u-bar^{t+1}
#                                                        (gather adjoint kernel)
#               u-bar^{t-1} += -u-bar^{t+1} on B           (the u_2 partial, -1)
# States are recomputed segment by segment from checkpoints (u^s, u^{s-1})
# stored every K steps: memory (2 T/K + K) states instead of T.
def time_loop_forward(n, T, D, c, u0, u1, store=None):
    """Returns u^T; store(t, u^t) is called for t = 0..T."""
    fam = "wave3d_r4"
    prev, cur = u0, u1
    if store:
        store(0, prev)
        store(1, cur)
    for t in range(1, T):
        nxt = torch.zeros_like(cur)
        api.primal(fam, n, {"D": D}, {"c": c, "u_1": cur, "u_2": prev, "u": nxt})
        prev, cur = cur, nxt
        if store:
            store(t + 1, cur)
    return cur


def time_loop_adjoint(n, T, D, c, u0, u1, w, checkpoint_every=None, fused=True,
                      workspace=None):
    """Gradient of J = <w, u^T> w.r.t. (u^0, u^1, c) through T-1 primal steps.
    Returns (u0_b, u1_b, c_b, stats).  `workspace`: an optional caller-owned
    list of state buffers kept across calls (a solver evaluating gradients
    repeatedly keeps its state memory; the buffers are zero outside the box
    and need no re-zeroing)."""
    import math
    fam = "wave3d_r4"
    K = checkpoint_every or max(1, int(math.isqrt(T)))
    lo, hi = 4, n - 5
    # state buffers: the primal writes only the box, so a buffer this driver
    # allocated (zero outside the box) can be reused without re-zeroing; the
    # caller's u0 / u1 are read, never written or recycled
    pool = [t for t in (workspace or []) if t.shape == u1.shape and t.dtype == u1.dtype
            and t.device == u1.device]
    if workspace is not None:
        workspace.clear()
    owned = {id(t): t for t in pool}

    def fresh():
        if pool:
            return pool.pop()
        t = torch.zeros_like(u1)
        owned[id(t)] = t
        return t

    def release(t, keep):
        if id(t) in owned and not any(t is k for k in keep):
            pool.append(t)

    # forward sweep keeping only the checkpoint pairs (u^{s-1}, u^s) at
    # s = 1, 1+K, 1+2K, ... (s < T), by reference (they are never written)
    ckpt = {1: (u0, u1)}
    prev, cur = u0, u1
    for t in range(1, T):
        nxt = fresh()
        api.primal(fam, n, {"D": D}, {"c": c, "u_1": cur, "u_2": prev, "u": nxt})
        release(prev, [x for pair in ckpt.values() for x in pair])
        prev, cur = cur, nxt
        s = t + 1
        if (s - 1) % K == 0 and s < T:
            ckpt[s] = (prev, cur)
    recomputed = 0
    # reverse sweep
    ub_next = w.clone()                  # u-bar^{t+1}
    ub_cur = torch.zeros_like(w)         # u-bar^t
    ub_prev = torch.zeros_like(w)        # u-bar^{t-1} (fully overwritten each step)
    c_b = torch.zeros_like(c)
    starts = sorted(ckpt)
    keep = [x for pair in ckpt.values() for x in pair]
    for s in reversed(starts):
        t_end = min(s + K, T)            # segment steps t = s .. t_end-1
        states = {s - 1: ckpt[s][0], s: ckpt[s][1]}
        for t in range(s, t_end - 1):    # recompute u^{s+1} .. u^{t_end-1}
            nxt = fresh()
            api.primal(fam, n, {"D": D}, {"c": c, "u_1": states[t], "u_2": states[t - 1],
                                          "u": nxt})
            states[t + 1] = nxt
            recomputed += 1
        for t in reversed(range(s, t_end)):
            # gather adjoint of step t, and u-bar^{t-1} = -u-bar^{t+1} on B
            # (the u_2 partial), 0 elsewhere -- one fused pass unless `fused`
            # is off (then the gather and sgb_box_set, bitwise the same)
            arrs = {"c": c, "c_b": c_b, "u_1": states[t], "u_1_b": ub_cur, "u_b": ub_next}
            if fused and c.dtype == torch.float32:
                api.adjoint_time_step(n, {"D": D}, arrs, ub_prev)
            else:
                api.adjoint(fam, n, {"D": D}, arrs)
                api.box_set(ub_prev, ub_next, -1.0, n, lo, hi)
            ub_next, ub_cur, ub_prev = ub_cur, ub_prev, ub_next
        for t, st in states.items():
            release(st, keep)
    # after the loop: ub_next = u-bar^1, ub_cur = u-bar^0
    if workspace is not None:  # every state buffer back to the caller's workspace
        workspace.extend(owned.values())
    stats = {"checkpoint_every": K, "checkpoints": len(starts), "recomputed_steps": recomputed,
             "adjoint_steps": T - 1}
    return ub_cur, ub_next, c_b, stats
