"""Multi-step drivers (cfg 5 independent steps, cfg 2 carried steps) against the
oracle, and the interior/edge split used to overlap the halo exchange.

Parity protocol: cfg 5 -- the whole multi-step run per
point and in the norm at 1e-5 (fp32 vs the fp64 oracle on the same fp32
inputs); cfg 2 -- norm <= 1e-5 over the carried run, per-point reported with a
looser gate (cancellation near zero crossings in fp32 accumulators).
"""
import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import torch
    assert torch.cuda.is_available()
    from paper_1907_02818_b200 import api, drivers
    return torch, api, drivers


def _np(t):
    return t.detach().to("cpu").double().numpy()


def test_cfg5_independent_steps_match_oracle(mods):
    torch, api, drivers = mods
    n, steps, seed, D = 28, 6, 3, 0.01
    arrays = drivers.run_independent(n, steps, seed=seed, D=D)
    got = _np(arrays["c_b"])
    c = _np(arrays["c"])
    scratch = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
    cb = np.zeros((n, n, n))
    for t in range(steps):
        drivers.regen_state(scratch, n, t, seed, 4)
        u1 = _np(scratch)
        drivers.regen_seed(scratch, n, t, seed)
        ub = _np(scratch)
        grids = {"c": c.copy(), "u_1": u1, "u_2": np.zeros_like(u1), "u": np.zeros_like(u1)}
        adjs = {"c_b": cb, "u_1_b": np.zeros_like(u1), "u_b": ub}
        assert oracle.run_program("wave3d_r4", n, {"D": D}, grids, adjs) == 0
        cb = adjs["c_b"]
    assert oracle.max_rel_err(got, cb) <= 1e-5
    assert oracle.norm_rel_err(got, cb) <= 1e-5


def test_cfg2_carried_steps_match_oracle(mods):
    torch, api, drivers = mods
    n, steps, seed, D = 20, 10, 5, 0.1
    arrays = drivers.run_carried(n, steps, seed=seed, D=D)
    c = _np(arrays["c"])
    scratch = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
    drivers.regen_seed(scratch, n, steps, seed)
    seedv = _np(scratch)
    u1b = np.zeros((n, n, n))
    u2b = np.zeros((n, n, n))
    cb = np.zeros((n, n, n))
    for t in reversed(range(steps)):
        drivers.regen_state(scratch, n, t, seed, 1)
        grids = {"c": c.copy(), "u_1": _np(scratch), "u_2": np.zeros((n, n, n)),
                 "u": np.zeros((n, n, n))}
        adjs = {"c_b": cb, "u_1_b": u1b, "u_2_b": u2b, "u_b": seedv}
        assert oracle.run_program("wave3d_c", n, {"D": D}, grids, adjs) == 0
        seedv, u1b, u2b, cb = adjs["u_1_b"], adjs["u_2_b"], np.zeros((n, n, n)), adjs["c_b"]
    for name, want in (("c_b", cb), ("u_b", seedv), ("u_1_b", u1b), ("u_2_b", u2b)):
        got = _np(arrays[name])
        assert oracle.norm_rel_err(got, want) <= 1e-5, name
        assert oracle.max_rel_err(got, want) <= 1e-5, name
    # the full-size (512^3) protocol against the reference's own emitted code
    # is tests/test_protocol_gpu.py::test_cfg2_carried_512


@pytest.mark.parametrize("n", [128, 256])
def test_run_carried_fused_equals_unfused_sweep(mods, n):
    """drivers.run_carried (u_2_b zeroing fused into every step's gather) is
    bitwise the plain sweep: accumulating gather, rotate, zero u_2_b."""
    torch, api, drivers = mods
    steps, seed, D = 10, 3, 0.1
    a = drivers.run_carried(n, steps, seed=seed, D=D)
    b = drivers.alloc("wave3d_c", n)
    drivers.init_static("wave3d_c", b, n, seed)
    drivers.regen_seed(b["u_b"], n, steps, seed)
    for t in reversed(range(steps)):
        drivers.regen_state(b["u_1"], n, t, seed, 1)
        api.adjoint("wave3d_c", n, {"D": D}, b)
        b["u_b"], b["u_1_b"], b["u_2_b"] = b["u_1_b"], b["u_2_b"], b["u_b"]
        b["u_2_b"].zero_()
    torch.cuda.synchronize()
    for k in ("c_b", "u_b", "u_1_b", "u_2_b"):
        assert torch.equal(a[k].view(torch.int32), b[k].view(torch.int32)), k
    # caller-supplied accumulators are kept: a non-zero u_2_b is accumulated into
    c = drivers.alloc("wave3d_c", n)
    drivers.init_static("wave3d_c", c, n, seed)
    drivers.regen_seed(c["u_b"], n, 1, seed)
    c["u_2_b"].fill_(1.0)
    d = {k: v.clone() for k, v in c.items()}
    drivers.run_carried(n, 1, seed=seed, D=D, arrays=c)
    drivers.regen_state(d["u_1"], n, 0, seed, 1)
    api.adjoint("wave3d_c", n, {"D": D}, d)
    torch.cuda.synchronize()
    assert torch.equal(c["u_b"], d["u_1_b"]) and torch.equal(c["u_1_b"], d["u_2_b"])


@pytest.mark.parametrize("family,n,world", [("wave3d_r4", 48, 2), ("wave3d_r4", 68, 3),
                                            ("wave3d_c", 40, 4)])
def test_interior_edge_split_equals_single_launch(mods, family, n, world):
    """The overlapped step computes interior planes, then the two edge bands in
    separate launches; per slab that must equal one launch over all owned planes."""
    torch, api, drivers = mods
    from paper_1907_02818_b200 import slab as slabmod
    from tests import inputs as gen
    scalars, grids, adjs = gen.family_inputs(family, n, seed=2, accumulate=True)
    dev = {k: torch.from_numpy(v.astype(np.float32)).cuda() for k, v in {**grids, **adjs}.items()}
    for r in range(world):
        sl = slabmod.decompose(n, oracle.family(family).radius, world, r)
        loc = {k: v[sl.base:sl.base + sl.nplanes].clone() for k, v in dev.items()}
        one = {k: v.clone() for k, v in loc.items()}
        api.adjoint_slab(family, n, scalars, one, sl.base, sl.nplanes, sl.own0, sl.own1)
        R = sl.radius
        lo_in = sl.own0 + (R if r > 0 else 0)
        hi_in = sl.own1 - (R if r < world - 1 else 0)
        api.adjoint_slab(family, n, scalars, loc, sl.base, sl.nplanes, lo_in, hi_in)
        if lo_in > sl.own0:
            api.adjoint_slab(family, n, scalars, loc, sl.base, sl.nplanes, sl.own0, lo_in)
        if hi_in < sl.own1:
            api.adjoint_slab(family, n, scalars, loc, sl.base, sl.nplanes, hi_in, sl.own1)
        torch.cuda.synchronize()
        for k in adjs:
            assert torch.equal(loc[k], one[k]), (family, r, k)


@pytest.mark.parametrize("n,world,regen,fresh", [(40, 2, True, False), (52, 3, True, True),
                                                 (40, 2, False, False), (44, 4, False, False),
                                                 (48, 2, True, True)])
def test_halo_prefetch_pipeline_bitwise(mods, n, world, regen, fresh):
    """HaloPrefetch (exchange of step t+1's halos on a side stream behind step
    t's compute, double-buffered u_1 / u_b) on emulated ranks of one GPU:
    every rank's owned planes of c_b / u_1_b after T steps are bitwise the
    single-GPU run's.  Each rank's regeneration writes its owned planes only
    (halo planes poisoned with NaN), and the emulated exchange fills the halo
    planes from the step's global field, so a step that read a set before its
    exchange, or a set already overwritten for a later step, shows up as
    NaN or as a wrong step's values."""
    torch, api, drivers = mods
    from paper_1907_02818_b200 import slab as slabmod
    fam, seed, D, T, R = "wave3d_r4", 5, 0.01, 5, 4
    sc = {"D": D}
    full = drivers.alloc(fam, n)
    drivers.init_static(fam, full, n, seed)
    api.fill_normal3d(full["u_1"], n, R, seed, 1)   # static inputs (cfg 4 style)
    api.fill_normal3d(full["u_b"], n, 0, seed, 3)
    static = {k: full[k].clone() for k in ("u_1", "u_b")}
    for t in range(T):
        if regen:
            drivers.regen_state(full["u_1"], n, t, seed, R)
            drivers.regen_seed(full["u_b"], n, t, seed)
            full["u_1_b"].zero_()
        api.adjoint(fam, n, sc, full)
    nan = float("nan")
    for r in range(world):
        sl = slabmod.decompose(n, R, world, r)
        loc = drivers.alloc(fam, n, sl)
        drivers.init_static(fam, loc, n, seed, sl)
        scratch = {k: torch.empty((n, n, n), device="cuda") for k in ("u_1", "u_b")}
        step_of = [0]
        top = sl.halo_lo + sl.owned

        def poison(t_):
            t_[:sl.halo_lo] = nan
            t_[top:] = nan

        for k in ("u_1", "u_b"):
            loc[k].copy_(static[k][sl.base:sl.base + sl.nplanes])
            poison(loc[k])

        def regen_fn(fs, t, sl=sl, step_of=step_of):
            drivers.regen_state(fs["u_1"], n, t, seed, R, sl)
            drivers.regen_seed(fs["u_b"], n, t, seed, sl)
            for k in fs:
                poison(fs[k])
            step_of[0] = t

        def exchange_fn(ts, sl=sl, step_of=step_of, scratch=scratch):
            if regen:
                drivers.regen_state(scratch["u_1"], n, step_of[0], seed, R)
                drivers.regen_seed(scratch["u_b"], n, step_of[0], seed)
                src = [scratch["u_1"], scratch["u_b"]]
            else:
                src = [static["u_1"], static["u_b"]]
            for dst, g in zip(ts, src):
                dst[:sl.halo_lo].copy_(g[sl.base:sl.own0])
                dst[top:].copy_(g[sl.own1:sl.base + sl.nplanes])

        pf = drivers.HaloPrefetch(fam, n, sc, loc, sl, regen=regen_fn if regen else None,
                                  exchange=exchange_fn, fresh=fresh)
        for t in range(T):
            if regen and not fresh:
                loc["u_1_b"].zero_()
            pf.step(t)
        torch.cuda.synchronize()
        own = slice(sl.halo_lo, top)
        for k in ("c_b", "u_1_b"):
            assert torch.equal(loc[k][own], full[k][sl.own0:sl.own1]), (r, k)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("noubwin", ["", "1"])
@pytest.mark.parametrize("n,world", [(40, 1), (68, 1), (37, 1), (48, 2), (68, 3), (36, 4)])
def test_fresh_gather_equals_zero_then_accumulate(mods, n, world, noubwin, dtype, sgbopt):
    """wave3d_r4_b_fresh(_slab)_{f32,f64} (u_1_b = this call's adjoint; the
    zeroing fused into the streaming kernels' MODE 4) is bitwise the zeroed
    u_1_b followed by the accumulating gather, c_b accumulated as usual --
    full grid (n = 37: the entry's memset + gather path) and every rank of
    z-slab decompositions, incl. the overlapped interior / edge-band split."""
    torch, api, drivers = mods
    from paper_1907_02818_b200 import slab as slabmod
    if noubwin:  # the in-kernel seed mask instead of the windowed seed map
        sgbopt.setenv("SGB_NO_UBWIN", "1")
    else:  # the L2-prefetching schedule gives the same bits
        sgbopt.setenv("SGB_V7_PREFETCH", "1")
    fam, sc = "wave3d_r4", {"D": 0.01}
    td, ti = (torch.float32, torch.int32) if dtype == "f32" else (torch.float64, torch.int64)
    g = torch.Generator(device="cpu").manual_seed(n + world)
    full = {k: torch.randn((n, n, n), generator=g).to(td).cuda()
            for k in ("c", "c_b", "u_1", "u_1_b", "u_b")}
    for r in range(world):
        sl = slabmod.decompose(n, 4, world, r) if world > 1 else None
        if sl is None:
            a = {k: v.clone() for k, v in full.items()}
        else:
            a = {k: v[sl.base:sl.base + sl.nplanes].clone() for k, v in full.items()}
        b = {k: v.clone() for k, v in a.items()}
        a["u_1_b"].fill_(float("nan"))  # every output plane must be written
        if sl is None:
            api.adjoint_fresh(fam, n, sc, a)
            b["u_1_b"].zero_()
            api.adjoint(fam, n, sc, b)
            own = slice(0, n)
        else:
            R = 4
            lo_in = sl.own0 + (R if r > 0 else 0)
            hi_in = sl.own1 - (R if r < world - 1 else 0)
            for (o0, o1) in ((lo_in, hi_in), (sl.own0, lo_in), (hi_in, sl.own1)):
                if o1 > o0:
                    api.adjoint_slab_fresh(fam, n, sc, a, sl.base, sl.nplanes, o0, o1)
            b["u_1_b"][sl.own0 - sl.base:sl.own1 - sl.base].zero_()
            api.adjoint_slab(fam, n, sc, b, sl.base, sl.nplanes, sl.own0, sl.own1)
            own = slice(sl.own0 - sl.base, sl.own1 - sl.base)
        torch.cuda.synchronize()
        for k in ("c_b", "u_1_b"):
            assert torch.equal(a[k][own].view(ti), b[k][own].view(ti)), (r, k)


@pytest.mark.parametrize("family", ["wave3d_c", "wave3d_c2"])
@pytest.mark.parametrize("n", [40, 68, 37])
def test_fresh_u2_gather_equals_zero_then_accumulate(mods, family, n):
    """wave3d_c(2)_b_fresh_u2_f32 (u_2_b written as the call's u_2 partial;
    the carried sweep's zeroing fused into the radius-1 streaming kernel) is
    bitwise the zeroed u_2_b followed by the accumulating gather, on every
    point incl. zero signs; n = 37 takes the entry's memset + gather path."""
    torch, api, drivers = mods
    sc = {"D": 0.1}
    g = torch.Generator(device="cpu").manual_seed(n + 7)
    a = {k: torch.randn((n, n, n), generator=g).cuda()
         for k in ("c", "c_b", "u_1", "u_1_b", "u_2_b", "u_b")}
    b = {k: v.clone() for k, v in a.items()}
    a["u_2_b"].fill_(float("nan"))
    api.adjoint_fresh_u2(family, n, sc, a)
    b["u_2_b"].zero_()
    api.adjoint(family, n, sc, b)
    torch.cuda.synchronize()
    for k in ("c_b", "u_1_b", "u_2_b"):
        assert torch.equal(a[k].view(torch.int32), b[k].view(torch.int32)), k


def test_generators_are_decomposition_invariant(mods):
    """fill_normal3d / fill_random / fill_layered values depend only on the
    global index: a slab regenerates exactly the single-GPU planes."""
    torch, api, drivers = mods
    n = 36
    full = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
    api.fill_normal3d(full, n, 4, 7, 11)
    flat = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
    api.fill_random(flat, 0, 7, 11, "normal", 0.0, 1.0)
    api.zero_halo(flat.view(n, n, n), 3, n, 4)
    assert torch.equal(full, flat.view(n, n, n))
    part = torch.empty((10, n, n), dtype=torch.float32, device="cuda")
    api.fill_normal3d(part, n, 4, 7, 11, 13, 10)
    assert torch.equal(part, full[13:23])
    lay = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
    api.fill_layered(lay, n, 8, 1.5, 4.5, 3)
    lpart = torch.empty((5, n, n), dtype=torch.float32, device="cuda")
    api.fill_layered(lpart, n, 8, 1.5, 4.5, 3, 30, 5)
    assert torch.equal(lpart, lay[30:35])
    z = full[4:-4, 4:-4, 4:-4]
    assert abs(float(z.mean())) < 0.05 and abs(float(z.std()) - 1) < 0.05


def test_time_loop_adjoint_checkpointing_and_gradient(mods):
    """adjoint of a whole wave3d_r4 time loop with forward
    recomputation from checkpoints.  Checkpoint spacing does not change the
    result (bitwise), and <grad, v> matches a central finite difference of
    J = <w, u^T> (fp64, the reference's dot-product test idea,
    interp.cpp:300-381, applied to the whole loop)."""
    torch, api, drivers = mods
    n, T, D = 20, 7, 0.01
    g = torch.Generator(device="cpu").manual_seed(3)

    def rnd(halo=4):
        x = torch.randn((n, n, n), generator=g, dtype=torch.float64)
        if halo:
            x[:halo] = 0; x[-halo:] = 0; x[:, :halo] = 0; x[:, -halo:] = 0
            x[:, :, :halo] = 0; x[:, :, -halo:] = 0
        return x.cuda()
    c = (torch.rand((n, n, n), generator=g, dtype=torch.float64) * 3 + 1.5).cuda()
    u0, u1, w = rnd(), rnd(), rnd(0)
    res = {}
    for K in (1, 2, 3, T):
        u0b, u1b, cb, st = drivers.time_loop_adjoint(n, T, D, c, u0, u1, w, checkpoint_every=K)
        res[K] = (u0b.clone(), u1b.clone(), cb.clone())
    for K in (2, 3, T):
        for a, b in zip(res[1], res[K]):
            assert torch.equal(a, b), K
    u0b, u1b, cb = res[3]

    def J(a0, a1, cc):
        return float((w * drivers.time_loop_forward(n, T, D, cc, a0, a1)).sum())
    v0, v1, vc = rnd(), rnd(), rnd()
    h = 1e-6
    fd = (J(u0 + h * v0, u1 + h * v1, c + h * vc) - J(u0 - h * v0, u1 - h * v1, c - h * vc)) / (2 * h)
    ad = float((v0 * u0b).sum() + (v1 * u1b).sum() + (vc * cb).sum())
    assert abs(fd - ad) / (1 + abs(ad)) < 1e-6, (fd, ad)


@pytest.mark.parametrize("noubwin", ["", "1"])
@pytest.mark.parametrize("n", [40, 68, 37])
def test_time_loop_fused_step_bitwise(mods, n, noubwin, sgbopt):
    """fp32 time loop: the fused reverse step (gather adjoint + u_2 partial in
    one radius-4 streaming pass, sgb_wave3d_r4_b_step_f32) equals the gather
    followed by sgb_box_set bit for bit -- the whole gradient after T steps,
    incl. the zeros outside the box; n = 37 takes the entry's two-launch path."""
    torch, api, drivers = mods
    if noubwin:  # the in-kernel seed mask instead of the windowed seed map
        sgbopt.setenv("SGB_NO_UBWIN", "1")
    T, D = 6, 0.01
    g = torch.Generator(device="cpu").manual_seed(n)
    c = (torch.rand((n, n, n), generator=g) * 3 + 1.5).cuda()
    u0, u1, w = (torch.randn((n, n, n), generator=g).cuda() for _ in range(3))
    a = drivers.time_loop_adjoint(n, T, D, c, u0, u1, w, checkpoint_every=2, fused=True)
    b = drivers.time_loop_adjoint(n, T, D, c, u0, u1, w, checkpoint_every=2, fused=False)
    for x, y in zip(a[:3], b[:3]):
        assert torch.equal(x, y)
    # a workspace kept across calls (reused state buffers) changes nothing
    ws = []
    for _ in range(2):
        r = drivers.time_loop_adjoint(n, T, D, c, u0, u1, w, checkpoint_every=2, workspace=ws)
        for x, y in zip(a[:3], r[:3]):
            assert torch.equal(x, y)
    assert ws
    # one step against the two-launch form, with a poisoned u_2_b buffer
    arrs = {"c": c, "c_b": torch.randn_like(c), "u_1": u1, "u_1_b": torch.randn_like(c),
            "u_b": w}
    ref = {k: v.clone() for k, v in arrs.items()}
    u2 = torch.full_like(c, float("nan"))
    api.adjoint_time_step(n, {"D": D}, arrs, u2)
    api.adjoint("wave3d_r4", n, {"D": D}, ref)
    u2_ref = torch.empty_like(c)
    api.box_set(u2_ref, w, -1.0, n, 4, n - 5)
    for k in ("c_b", "u_1_b"):
        assert torch.equal(arrs[k], ref[k]), k
    assert torch.equal(u2, u2_ref)
    assert torch.equal(u2.view(torch.int32), u2_ref.view(torch.int32))  # zero signs too


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("n,lo,hi,base,npl", [(40, 4, 35, 0, 40), (37, 1, 35, 0, 37),
                                              (64, 4, 59, 10, 30), (33, 3, 30, 5, 9)])
def test_box_axpy_matches_numpy(mods, n, lo, hi, base, npl, dtype):
    """y[B] += a * x[B] on a slab of planes, box edges and slab offsets that
    break 16-byte alignment included (vector and element paths)."""
    torch, api, _ = mods
    dt = torch.float32 if dtype == "f32" else torch.float64
    g = torch.Generator(device="cpu").manual_seed(n + lo)
    y = torch.randn(npl, n, n, generator=g, dtype=dt)
    x = torch.randn(npl, n, n, generator=g, dtype=dt)
    want = y.clone()
    for li in range(npl):
        i = base + li
        if lo <= i <= hi:
            want[li, lo:hi + 1, lo:hi + 1] += -0.5 * x[li, lo:hi + 1, lo:hi + 1]
    yd, xd = y.cuda(), x.cuda()
    api.box_axpy(yd, xd, -0.5, n, lo, hi, base, npl)
    torch.cuda.synchronize()
    assert torch.allclose(yd.cpu(), want, rtol=0, atol=1e-6 if dtype == "f32" else 1e-14)


@pytest.mark.parametrize("n", [64, 37])
def test_fill_normal3d_equals_elementwise_draw(mods, n):
    """The pairwise 3D generator (each Box-Muller pair computed once) yields
    exactly the values of the element-wise generator at the same global
    indices (odd n exercises the unpaired path)."""
    torch, api, _ = mods
    a = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    api.fill_normal3d(a, n, 0, 5, 3)
    api.fill_random(b, 0, 5, 3, "normal", 0.0, 1.0)
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("n,dtype", [(64, "f32"), (64, "f64"), (72, "f64"), (36, "f32"), (30, "f32"),
                                     (37, "f64")])
def test_fill_normal3d_pair_equals_two_fills(mods, n, dtype):
    """sgb_fill_normal3d_pair (cfg 5's regeneration of u_1 and the seed in one
    pass) writes bitwise the values of two fill_normal3d calls -- full grids
    and slabs, zero shells 4 / 0 / 1, mean and scale != (0, 1) -- on the fused
    fast path (n % 4 == 0) and the two-pass fallback (n % 4 != 0)."""
    torch, api, drivers = mods
    td = torch.float32 if dtype == "f32" else torch.float64
    for (i0, npl), (ha, hb), (mean, scale) in [((0, n), (4, 0), (0.0, 1.0)),
                                               ((5, 11), (1, 4), (0.25, 2.0)),
                                               ((n - 7, 7), (0, 0), (-1.0, 0.5))]:
        a = torch.full((npl, n, n), float("nan"), dtype=td, device="cuda")
        b = torch.full_like(a, float("nan"))
        api.fill_normal3d_pair(a, ha, 17, b, hb, 18, n, 9, i0, npl, mean, scale)
        wa, wb = torch.empty_like(a), torch.empty_like(a)
        api.fill_normal3d(wa, n, ha, 9, 17, i0, npl, mean, scale)
        api.fill_normal3d(wb, n, hb, 9, 18, i0, npl, mean, scale)
        torch.cuda.synchronize()
        assert torch.equal(a, wa) and torch.equal(b, wb), (i0, npl, ha, hb)


def test_regen_step_equals_state_and_seed(mods):
    """drivers.regen_step = regen_state + regen_seed, bitwise, on a slab too."""
    torch, api, drivers = mods
    from paper_1907_02818_b200 import slab as slabmod
    n = 48
    for sl in (None, slabmod.Slab(n, 4, 1, 3, 16, 32, 12, 24)):
        npl = n if sl is None else sl.nplanes
        a = torch.empty((npl, n, n), dtype=torch.float32, device="cuda")
        b, wa, wb = torch.empty_like(a), torch.empty_like(a), torch.empty_like(a)
        drivers.regen_step(a, b, n, 3, 0, 4, sl)
        drivers.regen_state(wa, n, 3, 0, 4, sl)
        drivers.regen_seed(wb, n, 3, 0, sl)
        torch.cuda.synchronize()
        assert torch.equal(a, wa) and torch.equal(b, wb)


def test_normal_generator_distribution(mods):
    """N(0, 1) at 2^26 samples: mean, variance, kurtosis and tail mass within
    a few standard errors; the (lg2, Fibonacci-lattice angle) pair has no
    correlation between its cos and sin branches."""
    torch, api, _ = mods
    n = 256
    a = torch.empty((n, n, n), dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    api.fill_normal3d_pair(a, 0, 1, b, 0, 2, n, 0)
    for x in (a, b):
        z = x.double().flatten()
        N = z.numel()
        m, v = float(z.mean()), float(z.var())
        k = float(((z - m) ** 4).mean()) / v ** 2
        assert abs(m) < 5 / N ** 0.5 and abs(v - 1) < 5 * (2 / N) ** 0.5, (m, v)
        assert abs(k - 3) < 5 * (24 / N) ** 0.5, k
        tail = float((z.abs() > 3).double().mean())
        assert abs(tail - 0.0026998) < 5 * (0.0027 / N) ** 0.5, tail
        assert float(z.abs().max()) > 5.0
        even, odd = z[0::2], z[1::2]
        assert abs(float((even * odd).mean())) < 5 / (N / 2) ** 0.5


@pytest.mark.parametrize("n", [72, 200, 520])
@pytest.mark.parametrize("fresh", [False, True])
def test_v8_interior_bitwise_equals_v7(mods, n, fresh, sgbopt):
    """The 4-rows-per-thread interior kernel (v8; default for the fresh form
    at n >= 512) forms every term in v7's order: bitwise the same c_b and
    u_1_b, accumulating and fresh."""
    torch, api, drivers = mods
    fam, sc = "wave3d_r4", {"D": 0.01}
    g = torch.Generator(device="cpu").manual_seed(n)
    base = {k: torch.randn((n, n, n), generator=g).cuda()
            for k in ("c", "c_b", "u_1", "u_1_b", "u_b")}
    out = {}
    for v8 in ("0", "1"):
        sgbopt.setenv("SGB_V8_INTERIOR", v8)
        a = {k: v.clone() for k, v in base.items()}
        (api.adjoint_fresh if fresh else api.adjoint)(fam, n, sc, a)
        torch.cuda.synchronize()
        out[v8] = a
    for k in ("c_b", "u_1_b"):
        assert torch.equal(out["0"][k].view(torch.int32), out["1"][k].view(torch.int32)), k


@pytest.mark.parametrize("fresh", [False, True])
def test_v8_balanced_last_wave_bitwise_equal(mods, fresh, sgbopt):
    """star3_v8_balanced (the interior launch when one chunk per column leaves
    a partly filled last wave: the remaining tiles' columns split between one
    CTA each and filler CTAs that walk several tiles, re-arming their
    mbarriers) computes the plain launch's bits -- automatic and forced split
    points, against the plain v8 launch and v7.  n = 704: 180 interior tiles on
    148 SMs with SGB_ICHUNKS=1 (cfg 5's 1024^3 takes this path by itself)."""
    torch, api, drivers = mods
    n, fam, sc = 704, "wave3d_r4", {"D": 0.01}
    g = torch.Generator(device="cuda").manual_seed(n)
    base = {k: torch.randn((n, n, n), generator=g, device="cuda")
            for k in ("c", "c_b", "u_1", "u_1_b", "u_b")}
    out = {}
    for name, env in (("v7", {"SGB_V8_INTERIOR": "0"}),
                      ("plain", {"SGB_V8_INTERIOR": "1", "SGB_V8_BALANCE": "0"}),
                      ("auto", {"SGB_V8_INTERIOR": "1", "SGB_V8_BALANCE": "1"}),
                      ("m100", {"SGB_V8_INTERIOR": "1", "SGB_V8_BALANCE": "100"}),
                      ("m500", {"SGB_V8_INTERIOR": "1", "SGB_V8_BALANCE": "500"})):
        with sgbopt.context() as m:
            m.setenv("SGB_ICHUNKS", "1")
            for k, v in env.items():
                m.setenv(k, v)
            a = {k: t.clone() for k, t in base.items() if k in ("c_b", "u_1_b")}
            a.update({k: base[k] for k in ("c", "u_1", "u_b")})
            (api.adjoint_fresh if fresh else api.adjoint)(fam, n, sc, a)
            torch.cuda.synchronize()
        out[name] = {k: a[k] for k in ("c_b", "u_1_b")}
    for name in ("plain", "auto", "m100", "m500"):
        for k in ("c_b", "u_1_b"):
            assert torch.equal(out["v7"][k].view(torch.int32),
                               out[name][k].view(torch.int32)), (name, k)


@pytest.mark.parametrize("fresh", [False, True])
def test_f64_v8_bitwise_equals_two_row_form(mods, fresh, sgbopt):
    """The opt-in 4-rows-per-thread fp64 radius-4 kernel (SGB_F64_V8=1) forms
    every term in the 2-row kernel's order: bitwise the same result."""
    torch, api, drivers = mods
    n, fam, sc = 72, "wave3d_r4", {"D": 0.01}
    g = torch.Generator(device="cpu").manual_seed(3)
    base = {k: torch.randn((n, n, n), generator=g, dtype=torch.float64).cuda()
            for k in ("c", "c_b", "u_1", "u_1_b", "u_b")}
    out = {}
    for v in ("0", "1"):
        sgbopt.setenv("SGB_F64_V8", v)
        a = {k: t.clone() for k, t in base.items()}
        (api.adjoint_fresh if fresh else api.adjoint)(fam, n, sc, a)
        torch.cuda.synchronize()
        out[v] = a
    for k in ("c_b", "u_1_b"):
        assert torch.equal(out["0"][k].view(torch.int64), out["1"][k].view(torch.int64)), k


@pytest.mark.parametrize("n", [72, 200, 520])
@pytest.mark.parametrize("fresh", [False, True])
@pytest.mark.parametrize("opts", [{"SGB_V8_FRAME": "1"},
                                  {"SGB_V8_FRAME": "1", "SGB_ICHUNKS": "3", "SGB_ICHUNKS_F": "5"}])
def test_v8_frame_bitwise_equal_v7(mods, n, fresh, opts, sgbopt):
    """v8's frame body (per-point masks for 4 rows) gives v7's bits, full
    grids with partial tiles, any i-chunking."""
    torch, api, drivers = mods
    fam, sc = "wave3d_r4", {"D": 0.01}
    g = torch.Generator(device="cpu").manual_seed(n + 7)
    base = {k: torch.randn((n, n, n), generator=g).cuda()
            for k in ("c", "c_b", "u_1", "u_1_b", "u_b")}
    out = {}
    for variant in ("v7", "v8"):
        with sgbopt.context() as m:
            m.setenv("SGB_V8_INTERIOR", "1" if variant == "v8" else "0")
            if variant == "v8":
                for k, v in opts.items():
                    m.setenv(k, v)
            a = {k: t.clone() for k, t in base.items()}
            (api.adjoint_fresh if fresh else api.adjoint)(fam, n, sc, a)
            torch.cuda.synchronize()
        out[variant] = a
    for k in ("c_b", "u_1_b"):
        assert torch.equal(out["v7"][k].view(torch.int32), out["v8"][k].view(torch.int32)), k
