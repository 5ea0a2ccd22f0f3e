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
    for name, want in (("c_b", cb), ("u_b", seedv), ("u_1_b", u1b)):
        got = _np(arrays[name])
        assert oracle.norm_rel_err(got, want) <= 1e-5, name
        assert oracle.max_rel_err(got, want) <= 1e-4, name


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
