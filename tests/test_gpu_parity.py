"""GPU parity: the sm_100a kernels (through the C ABI) against the reference.

Tolerances (BASELINE.json north_star): fp64 per point |a-b|/(1+|b|) <= 1e-12
(compare_grids, interp.cpp:290-298); fp32 <= 1e-5 per point and in the norm,
against the fp64 oracle evaluated on the fp32-rounded inputs.  The oracle
(oracle/sg_oracle.c) is pinned to the reference by tests/test_oracle_pins.py;
the committed goldens are the reference's own outputs.
"""
import numpy as np
import pytest

from oracle import oracle
from tests import inputs as gen
from tests.test_oracle_pins import _golden_cases, load_golden

pytestmark = pytest.mark.gpu

GPU_FAMILIES = ("wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4")
TOL = {"f64": 1e-12, "f32": 1e-5}


@pytest.fixture(scope="module")
def api():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1907_02818_b200 import api as _api
    return _api


def _round(grids, dtype):
    if dtype == "f64":
        return {k: v.copy() for k, v in grids.items()}
    return {k: v.astype(np.float32).astype(np.float64) for k, v in grids.items()}


def oracle_gather(name, n, scalars, grids, adjs):
    out = {k: v.copy() for k, v in adjs.items()}
    assert oracle.run_program(name, n, scalars, {k: v.copy() for k, v in grids.items()}, out) == 0
    return out


def check_close(got, want, dtype, what):
    tol = TOL[dtype]
    e = oracle.max_rel_err(got, want)
    assert e <= tol, f"{what}: per-point {e:.3e} > {tol}"
    if dtype == "f32":
        ne = oracle.norm_rel_err(got, want)
        assert ne <= tol, f"{what}: norm {ne:.3e} > {tol}"


def gpu_cases():
    return [c for c in _golden_cases() if c.rsplit("_n", 1)[0] in GPU_FAMILIES]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("case", gpu_cases())
def test_gather_matches_reference_golden(api, case, dtype):
    name, n, f, scalars, grids, adjs, refs = load_golden(case)
    g, a = _round(grids, dtype), _round(adjs, dtype)
    got = api.run_program(name, n, scalars, g, a, dtype=dtype)
    for adj in got:
        if adj == f.seed:
            continue
        if dtype == "f64":
            check_close(got[adj], refs["gather_" + adj], dtype, adj)
        else:
            want = oracle_gather(name, n, scalars, g, a)
            check_close(got[adj], want[adj], dtype, adj)


@pytest.mark.parametrize("case", gpu_cases())
def test_primal_matches_reference_golden(api, case):
    name, n, f, scalars, grids, adjs, refs = load_golden(case)
    got = api.run_nest(name, n, scalars, grids, dtype="f64")
    out = f.arrays[f.output]
    check_close(got[out], refs["primal_" + out], "f64", "primal")


@pytest.mark.parametrize("case", gpu_cases())
def test_scatter_matches_reference_golden(api, case):
    name, n, f, scalars, grids, adjs, refs = load_golden(case)
    got = api.run_scatter_adjoint(name, n, scalars, grids, adjs, dtype="f64")
    for adj in got:
        if adj != f.seed:
            check_close(got[adj], refs["scatter_" + adj], "f64", adj)


# Sizes that exercise the TMA streaming kernel (n % 4 == 0, n >= 16), partial
# 64x16 tiles (n not a tile multiple) and the general per-point kernel (odd n).
SIZES = {
    "wave3d_r4": [17, 24, 36, 68, 97],
    "wave3d_c": [5, 16, 33, 40, 68],
    "wave3d_c2": [20, 41],
    "wave1d": [5, 1000, 4099],
    "burgers2d": [5, 64, 203, 300, 1030],
}


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("name,n", [(k, n) for k, v in SIZES.items() for n in v])
def test_gather_matches_oracle_sizes(api, name, n, dtype):
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n, accumulate=True)
    g, a = _round(grids, dtype), _round(adjs, dtype)
    got = api.run_program(name, n, scalars, g, a, dtype=dtype)
    want = oracle_gather(name, n, scalars, g, a)
    f = oracle.family(name)
    for adj in got:
        if adj != f.seed:
            check_close(got[adj], want[adj], dtype, f"{name} n={n} {adj}")


@pytest.mark.parametrize("name", GPU_FAMILIES)
def test_untouched_points_keep_their_bits(api, name):
    """Points no term reaches are left untouched: seed the
    adjoints with NaN and -0.0 there and check they survive bit for bit."""
    n = {"wave1d": 64, "burgers2d": 32, "wave3d_r4": 32}.get(name, 24)
    scalars, grids, adjs = gen.family_inputs(name, n, seed=3, accumulate=True)
    f = oracle.family(name)
    # reached mask from the oracle: run with zero adjoints and a seed of ones,
    # then mark every point some term writes (terms are dense nonzero here)
    probe = {k: np.zeros_like(v) for k, v in adjs.items()}
    probe[f.seed] = np.ones_like(adjs[f.seed])
    reached = {}
    for ti, (arr, off) in enumerate(f.terms):
        adj = f.adjoints[arr]
        m = reached.setdefault(adj, np.zeros(f.shape(n), bool))
        lo, hi = f.lo, n + f.hi_n
        sl = tuple(slice(lo + o, hi + o + 1) for o in off)
        m[sl] = True
    for dtype in ("f64", "f32"):
        a = _round(adjs, dtype)
        for adj, m in reached.items():
            a[adj][~m] = np.nan
            flat = np.flatnonzero(~m)
            if flat.size:
                a[adj].flat[flat[0]] = -0.0
        got = api.run_program(name, n, scalars, _round(grids, dtype), a, dtype=dtype)
        for adj, m in reached.items():
            before = a[adj][~m].astype(np.float32 if dtype == "f32" else np.float64)
            after = got[adj][~m].astype(before.dtype)
            assert np.array_equal(before.view(np.uint32 if dtype == "f32" else np.uint64),
                                  after.view(np.uint32 if dtype == "f32" else np.uint64)), adj
            assert np.all(np.isfinite(got[adj][m])), adj


@pytest.mark.parametrize("name,n", [("wave1d", 4), ("wave3d_c", 4), ("burgers2d", 4),
                                    ("wave3d_r4", 16)])
def test_guard_violation_returns_1_and_touches_nothing(api, name, n):
    from paper_1907_02818_b200 import _lib
    scalars, grids, adjs = gen.family_inputs(name, n, seed=1, accumulate=True)
    with pytest.raises(_lib.GuardViolation):
        api.run_program(name, n, scalars, grids, adjs, dtype="f64")


@pytest.mark.parametrize("name,n,nslabs", [("wave3d_r4", 40, 2), ("wave3d_r4", 68, 3),
                                           ("wave3d_r4", 37, 4), ("wave3d_c", 40, 4),
                                           ("wave3d_c", 19, 3)])
def test_slabs_reassemble_to_single_gpu_bitwise(api, name, n, nslabs):
    """z-slab decomposition: each slab holds its owned planes
    plus R halo planes; the union of slab outputs equals the single-GPU run."""
    import torch
    scalars, grids, adjs = gen.family_inputs(name, n, seed=11, accumulate=True)
    R = oracle.family(name).radius
    dev = {k: torch.from_numpy(v.astype(np.float32)).cuda() for k, v in {**grids, **adjs}.items()}
    full = {k: v.clone() for k, v in dev.items()}
    api.adjoint(name, n, scalars, full)
    bounds = np.linspace(0, n, nslabs + 1).astype(int)
    outs = {k: v.clone() for k, v in dev.items()}
    for s in range(nslabs):
        i0, i1 = int(bounds[s]), int(bounds[s + 1])
        a0, a1 = max(i0 - R, 0), min(i1 + R, n)
        loc = {k: v[a0:a1].contiguous() for k, v in dev.items()}
        api.adjoint_slab(name, n, scalars, loc, a0, a1 - a0, i0, i1)
        for k in adjs:
            outs[k][i0:i1] = loc[k][i0 - a0:i1 - a0]
    torch.cuda.synchronize()
    for k in adjs:
        assert torch.equal(outs[k], full[k]), k


def test_dot_product_test_on_gpu(api):
    """<(F(u+hv)-F(u-hv))/2h, w> == <v, J^T w> (dot_product_test,
    interp.cpp:300-381) with the GPU primal and GPU gather adjoint, fp64."""
    rng = np.random.default_rng(5)
    for name, n in [("wave1d", 257), ("wave3d_c", 20), ("wave3d_r4", 24), ("burgers2d", 64)]:
        f = oracle.family(name)
        scalars, grids, _ = gen.family_inputs(name, n, seed=9, ties=False)
        inputs = f.active_inputs
        out = f.arrays[f.output]
        v = {a: rng.standard_normal(grids[a].shape) for a in inputs}
        w = rng.standard_normal(grids[out].shape)
        umax = max(np.abs(grids[a]).max() for a in inputs)
        h = 1e-5 * (1 + umax)
        gp = {k: x.copy() for k, x in grids.items()}
        gm = {k: x.copy() for k, x in grids.items()}
        for a in inputs:
            gp[a] += h * v[a]
            gm[a] -= h * v[a]
        gp[out][:] = 0
        gm[out][:] = 0
        rp = api.run_nest(name, n, scalars, gp)[out]
        rm = api.run_nest(name, n, scalars, gm)[out]
        lhs = float(np.sum(w * (rp - rm) / (2 * h)))
        adjs = {f.adjoints[f.arrays.index(a)]: np.zeros(grids[a].shape) for a in inputs}
        adjs[f.seed] = w
        res = api.run_program(name, n, scalars, grids, adjs)
        rhs = float(sum(np.sum(v[a] * res[f.adjoints[f.arrays.index(a)]]) for a in inputs))
        err = abs(lhs - rhs) / (1 + abs(rhs))
        assert err <= 1e-4, (name, err)


@pytest.mark.parametrize("name,n,dtype", [("wave3d_r4", 136, "f32"), ("wave3d_c", 128, "f32"),
                                          ("wave3d_r4", 40, "f64"), ("wave3d_r4", 136, "f64"),
                                          ("wave3d_c", 130, "f64"), ("burgers2d", 64, "f64"),
                                          ("burgers2d", 1000, "f64"), ("burgers2d", 516, "f32"),
                                          ("wave1d", 300, "f64"), ("wave1d", 100002, "f64"),
                                          ("wave1d", 4099, "f64"), ("wave1d", 5000, "f32")])
def test_host_buffer_plan_entry(api, name, n, dtype):
    """sgb_plan_run_adjoint_host (host arrays in, accumulated adjoints out;
    pipelined over chunks of the outermost dimension for 3D fp32, burgers2d
    rows and wave1d index ranges; one shot otherwise) equals the
    device-pointer entry bit for bit."""
    import torch
    scalars, grids, adjs = gen.family_inputs(name, n, seed=4, accumulate=True)
    np_dt = np.float32 if dtype == "f32" else np.float64
    host = {k: np.ascontiguousarray(v.astype(np_dt)) for k, v in {**grids, **adjs}.items()}
    want = api.run_program(name, n, scalars, {k: host[k].astype(np.float64) for k in grids},
                           {k: host[k].astype(np.float64) for k in adjs}, dtype=dtype)
    plan = api.Plan(name, n, dtype)
    plan.run_adjoint_host(scalars, host)
    plan.close()
    f = oracle.family(name)
    for k in adjs:
        got = host[k].astype(np.float64)
        assert np.array_equal(got, want[k]), k


@pytest.mark.parametrize("n", [68, 97, 136])
def test_r4_launch_variants_bitwise_equal(api, n, sgbopt):
    """The radius-4 launch knobs (windowed seed map vs in-kernel mask, one
    launch vs interior/frame launches, wave-model vs forced i-chunking, frame
    on a side stream) change only scheduling: every
    point's arithmetic is the same, so the results are bitwise identical, and
    the default matches the oracle."""
    name = "wave3d_r4"
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n + 1, accumulate=True)
    g, a = _round(grids, "f32"), _round(adjs, "f32")
    base = api.run_program(name, n, scalars, g, a, dtype="f32")
    want = oracle_gather(name, n, scalars, g, a)
    for adj in ("c_b", "u_1_b"):
        check_close(base[adj], want[adj], "f32", f"{name} n={n} {adj}")
    for env in ({"SGB_NO_UBWIN": "1"}, {"SGB_ICHUNKS": "3", "SGB_ICHUNKS_F": "5"},
                {"SGB_ICHUNKS": "1", "SGB_ICHUNKS_F": "1"}, {"SGB_FORK": "1"},
                {"SGB_V7_UNIFIED": "1"}, {"SGB_V7_UNIFIED": "1", "SGB_ICHUNKS": "3"},
                {"SGB_V7_SPLIT": "1"}, {"SGB_FORK": "0"}, {"SGB_V7_PREFETCH": "2"}):
        with sgbopt.context() as m:
            for k, v in env.items():
                m.setenv(k, v)
            got = api.run_program(name, n, scalars, g, a, dtype="f32")
        for adj in ("c_b", "u_1_b"):
            assert np.array_equal(got[adj], base[adj]), (env, adj)


@pytest.mark.parametrize("name,n", [("wave3d_r4", 68), ("wave3d_r4", 136), ("wave3d_r4", 200),
                                    ("wave3d_c", 136)])
def test_primal_chunking_bitwise_equal(api, name, n, sgbopt):
    """The streaming primal's i-chunk count (default: ~48-plane chunks at
    radius 4, wave model at radius 1) changes only which CTA streams which
    planes: results are bitwise identical for any count, incl. one chunk per
    column and chunks shorter than the 2R halo."""
    scalars, grids, _ = gen.family_inputs(name, n, seed=n + 11)
    f = oracle.family(name)
    out = f.arrays[f.output]
    grids[out] = np.random.default_rng(n + 1).standard_normal(grids[out].shape)
    g = _round(grids, "f32")
    base = api.run_nest(name, n, scalars, g, dtype="f32")[out]
    for chunks in ("1", "2", "5", "64"):
        with sgbopt.context() as m:
            m.setenv("SGB_PRIMAL_CHUNKS", chunks)
            got = api.run_nest(name, n, scalars, g, dtype="f32")[out]
        assert np.array_equal(got, base), chunks


@pytest.mark.parametrize("n", [64, 300, 1030])
def test_burgers_ring_variants_bitwise_equal(api, n, sgbopt):
    """burgers2d ring kernel: stage count and rows per CTA change only the
    schedule, so results are bitwise identical; the register-streaming kernel
    it replaced agrees to fp64 rounding."""
    name = "burgers2d"
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n + 3, accumulate=True)
    base = api.run_program(name, n, scalars, grids, adjs, dtype="f64")
    want = oracle_gather(name, n, scalars, grids, adjs)
    check_close(base["u_1_b"], want["u_1_b"], "f64", f"{name} n={n}")
    for env in ({"SGB_BURGERS_RING_S": "4"}, {"SGB_BURGERS_RING_S": "8"},
                {"SGB_BURGERS_RING_RB": "7"}, {"SGB_BURGERS_RING_RB": "256"}):
        with sgbopt.context() as m:
            for k, v in env.items():
                m.setenv(k, v)
            got = api.run_program(name, n, scalars, grids, adjs, dtype="f64")
        assert np.array_equal(got["u_1_b"], base["u_1_b"]), env
    with sgbopt.context() as m:
        m.setenv("SGB_BURGERS_NORING", "1")
        old = api.run_program(name, n, scalars, grids, adjs, dtype="f64")
    assert oracle.max_rel_err(old["u_1_b"], base["u_1_b"]) <= 1e-14


@pytest.mark.parametrize("name,n", [("wave1d", 1000), ("wave3d_c", 36), ("wave3d_c2", 20),
                                    ("burgers2d", 300), ("wave3d_r4", 40)])
def test_verify_problem_equivalence_on_gpu(api, name, n):
    """verify_problem's oracle-equivalence half (interp.cpp:413-435) run on the
    B200: the GPU gather adjoint and the GPU atomic-scatter adjoint agree per
    point at 1e-12 (fp64) on every non-output active adjoint."""
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n + 5, accumulate=True)
    gat = api.run_program(name, n, scalars, grids, adjs, dtype="f64")
    sca = api.run_scatter_adjoint(name, n, scalars, grids, adjs, dtype="f64")
    f = oracle.family(name)
    for adj in gat:
        if adj != f.seed:
            e = oracle.max_rel_err(gat[adj], sca[adj])
            assert e <= 1e-12, (name, adj, e)


@pytest.mark.parametrize("name", ["wave3d_r4", "wave3d_c", "wave3d_c2"])
@pytest.mark.parametrize("n", [17, 24, 36, 68, 97, 136, 200])
def test_primal_f32_matches_oracle(api, name, n):
    """fp32 primal (TMA streaming kernel where n % 4 == 0, per-point kernel
    otherwise) against the oracle's run_nest on the fp32-rounded inputs; the
    output array starts non-zero, so '+=' families and the untouched points
    outside the primal box are checked too."""
    scalars, grids, _ = gen.family_inputs(name, n, seed=n + 7)
    f = oracle.family(name)
    out = f.arrays[f.output]
    grids[out] = np.random.default_rng(n).standard_normal(grids[out].shape)
    g = _round(grids, "f32")
    got = api.run_nest(name, n, scalars, g, dtype="f32")
    want = {k: v.copy() for k, v in g.items()}
    assert oracle.run_primal(name, n, scalars, want) == 0
    check_close(got[out], want[out], "f32", f"{name} n={n} primal")


@pytest.mark.parametrize("n", [20, 24, 40, 66, 98, 136])
def test_primal_f64_r4_streaming(api, n, sgbopt):
    """fp64 radius-4 streaming primal (even n): matches the oracle's run_nest
    at 1e-12 (the output starts non-zero, so points outside the box are
    checked to be untouched); i-chunking changes nothing (bitwise)."""
    name = "wave3d_r4"
    scalars, grids, _ = gen.family_inputs(name, n, seed=n + 17)
    f = oracle.family(name)
    out = f.arrays[f.output]
    grids[out] = np.random.default_rng(n + 3).standard_normal(grids[out].shape)
    got = api.run_nest(name, n, scalars, grids, dtype="f64")
    want = {k: v.copy() for k, v in grids.items()}
    assert oracle.run_primal(name, n, scalars, want) == 0
    check_close(got[out], want[out], "f64", f"{name} n={n} primal")
    assert np.array_equal(got[out][:4], grids[out][:4])  # planes outside the box untouched
    for chunks in ("1", "5"):
        with sgbopt.context() as m:
            m.setenv("SGB_PRIMAL_CHUNKS", chunks)
            again = api.run_nest(name, n, scalars, grids, dtype="f64")
        assert np.array_equal(again[out], got[out]), chunks


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n", [64, 300, 1032])
def test_burgers_primal_ring_variants_bitwise_equal(api, n, dtype, sgbopt):
    """The ring primal evaluates the register-streaming kernel's expression
    with the same grouping: bitwise equal to it, for every stage count and
    rows-per-CTA (incl. a strip taller than the grid)."""
    name = "burgers2d"
    scalars, grids, _ = gen.family_inputs(name, n, seed=n + 13)
    grids["u"] = np.random.default_rng(n + 2).standard_normal(grids["u"].shape)
    g = _round(grids, dtype)
    base = api.run_nest(name, n, scalars, g, dtype=dtype)["u"]
    for env in ({"SGB_BURGERS_NORING": "1"}, {"SGB_BURGERS_PRIMAL_S": "4"},
                {"SGB_BURGERS_PRIMAL_S": "8"}, {"SGB_BURGERS_PRIMAL_RB": "7"},
                {"SGB_BURGERS_PRIMAL_RB": "5000"}):
        with sgbopt.context() as m:
            for k, v in env.items():
                m.setenv(k, v)
            got = api.run_nest(name, n, scalars, g, dtype=dtype)["u"]
        assert np.array_equal(got, base), env


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n", [5, 64, 203, 300, 1030])
def test_burgers_primal_matches_oracle(api, n, dtype):
    """burgers2d primal (strip ring kernel where rows are 16-byte multiples,
    row-streaming kernel for other even n, per-point otherwise) against the
    oracle's run_nest; untouched ring keeps its values."""
    name = "burgers2d"
    scalars, grids, _ = gen.family_inputs(name, n, seed=n + 11)
    grids["u"] = np.random.default_rng(n).standard_normal(grids["u"].shape)
    g = _round(grids, dtype)
    got = api.run_nest(name, n, scalars, g, dtype=dtype)
    want = {k: v.copy() for k, v in g.items()}
    assert oracle.run_primal(name, n, scalars, want) == 0
    check_close(got["u"], want["u"], dtype, f"burgers2d n={n} primal")


def test_short_buffers_are_rejected(api):
    """A device array smaller than the grid is refused before any launch (the
    reference raises on out-of-bounds access) and nothing is written."""
    import torch
    from paper_1907_02818_b200 import _lib
    n = 24
    arrays = {nm: torch.zeros((n, n, n), device="cuda")
              for nm in api.array_params("wave3d_r4", "adjoint")}
    arrays["u_1_b"] = torch.zeros((n - 1, n, n), device="cuda")
    before = _lib.launch_count()
    with pytest.raises(_lib.StencilError):
        api.adjoint("wave3d_r4", n, {"D": 0.01}, arrays)
    assert _lib.launch_count() == before
    assert not arrays["c_b"].any()


@pytest.mark.parametrize("name,n,nslabs", [("wave3d_r4", 136, 3), ("wave3d_r4", 68, 2),
                                           ("wave3d_c", 128, 4)])
def test_slab_plans_reassemble_full_plan(api, name, n, nslabs):
    """sgb_plan_create_slab: each rank's host-buffer call on its local planes
    (owned + halos) returns the owned planes of the full-grid plan bit for bit."""
    from paper_1907_02818_b200 import slab
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n + 2, accumulate=True)
    host = {k: np.ascontiguousarray(v.astype(np.float32)) for k, v in {**grids, **adjs}.items()}
    names = api.array_params(name, "adjoint")
    full = {k: host[k].copy() for k in names}
    plan = api.Plan(name, n, "f32")
    plan.run_adjoint_host(scalars, full)
    plan.close()
    R = 4 if name == "wave3d_r4" else 1
    f = oracle.family(name)
    for rank in range(nslabs):
        sl = slab.decompose(n, R, nslabs, rank)
        loc = {k: np.ascontiguousarray(host[k][sl.base:sl.base + sl.nplanes]) for k in names}
        p = api.Plan(name, n, "f32", slab=sl)
        p.run_adjoint_host(scalars, loc)
        p.close()
        a, b = sl.own0 - sl.base, sl.own1 - sl.base
        for k in names:
            if k in adjs and k != f.seed:
                assert np.array_equal(loc[k][a:b], full[k][sl.own0:sl.own1]), (rank, k)


@pytest.mark.parametrize("n,dtype,nslabs", [(136, "f32", 1), (160, "f32", 1), (136, "f64", 1),
                                             (40, "f32", 1), (272, "f32", 2)])
def test_host_sweep_equals_per_step_calls(api, n, dtype, nslabs):
    """sgb_plan_sweep_* (c, c_b resident on the device for the whole reverse
    sweep; a step moves u_1, u_b in and its own adjoint u_1_b out) gives, bit
    for bit, what the caller of the reference ABI gets from zeroing u_1_b and
    calling the accumulating host entry once per step; the first step also
    against the oracle.  nslabs = 2: one rank's slab plan (halos in the host
    arrays) returns the owned planes of the full-grid sweep."""
    from paper_1907_02818_b200 import slab
    name, T = "wave3d_r4", 3
    np_dt = np.float32 if dtype == "f32" else np.float64
    names = api.array_params(name, "adjoint")
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n + 31, accumulate=True)
    c = np.ascontiguousarray(grids["c"].astype(np_dt))
    c_b0 = np.ascontiguousarray(adjs["c_b"].astype(np_dt))
    steps = []
    for t in range(T):
        _, g, a = gen.family_inputs(name, n, seed=1000 + 7 * t + n, accumulate=True)
        steps.append((np.ascontiguousarray(g["u_1"].astype(np_dt)),
                      np.ascontiguousarray(a["u_b"].astype(np_dt))))
    # per-step calls of the accumulating entry, u_1_b zeroed by the caller
    ref = {"c": c.copy(), "c_b": c_b0.copy()}
    want_u1b = []
    plan = api.Plan(name, n, dtype)
    for u_1, u_b in steps:
        ref.update(u_1=u_1.copy(), u_b=u_b.copy(), u_1_b=np.zeros_like(u_1))
        plan.run_adjoint_host(scalars, ref)
        want_u1b.append(ref["u_1_b"].copy())
    plan.close()
    ranks = [slab.decompose(n, 4, nslabs, r) for r in range(nslabs)] if nslabs > 1 else [None]
    for sl in ranks:
        loc = (lambda x: x) if sl is None else \
            (lambda x: np.ascontiguousarray(x[sl.base:sl.base + sl.nplanes]))
        own = slice(None) if sl is None else slice(sl.own0 - sl.base, sl.own1 - sl.base)
        gown = slice(None) if sl is None else slice(sl.own0, sl.own1)
        host = {"c": loc(c), "c_b": loc(c_b0).copy()}
        plan = api.Plan(name, n, dtype, slab=sl)
        with pytest.raises(api._lib.StencilError):
            plan.sweep_step_host(scalars, {"u_1": loc(steps[0][0]), "u_b": loc(steps[0][1]),
                                           "u_1_b": loc(steps[0][0]).copy()})
        plan.sweep_begin(host)
        for t, (u_1, u_b) in enumerate(steps):
            out = np.full_like(loc(u_1), np.nan)
            plan.sweep_step_host(scalars, {"u_1": loc(u_1), "u_b": loc(u_b), "u_1_b": out})
            assert np.array_equal(out[own], want_u1b[t][gown]), ("u_1_b", t)
        plan.sweep_end(host)
        plan.close()
        assert np.array_equal(host["c_b"][own], ref["c_b"][gown])
    # the first step against the oracle
    g0 = {"c": c.astype(np.float64), "u_1": steps[0][0].astype(np.float64)}
    a0 = {"c_b": c_b0.astype(np.float64), "u_1_b": np.zeros((n, n, n)),
          "u_b": steps[0][1].astype(np.float64)}
    want = oracle_gather(name, n, scalars, g0, a0)
    check_close(want_u1b[0].astype(np.float64), want["u_1_b"], dtype, "sweep step 0 u_1_b")


def test_host_sweep_refuses_other_families(api):
    for fam, n, dt in (("burgers2d", 64, "f64"), ("wave3d_c2", 32, "f32")):
        plan = api.Plan(fam, n, dt)
        with pytest.raises(api._lib.StencilError):
            plan.sweep_begin({})
        plan.close()


@pytest.mark.parametrize("n,dtype", [(132, "f32"), (64, "f32"), (40, "f64")])
def test_host_carried_sweep_equals_per_step_calls(api, n, dtype):
    """sgb_plan_sweep_* on a wave3d_c plan (BASELINE cfg 2's carried steps with
    host-held states): c, c_b and the adjoints stay on the device, a step moves
    only u_1 in and rotates seed <- u_1_b, u_1_b <- u_2_b, u_2_b <- 0 there.
    Bit for bit what a caller of the reference ABI gets from the accumulating
    host entry per step followed by the same rotation of its host arrays."""
    name, T = "wave3d_c", 4
    np_dt = np.float32 if dtype == "f32" else np.float64
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n + 77, accumulate=True)
    cast = lambda x: np.ascontiguousarray(x.astype(np_dt))  # noqa: E731
    states = []
    for t in range(T):
        _, g, _ = gen.family_inputs(name, n, seed=500 + 11 * t + n, accumulate=True)
        states.append(cast(g["u_1"]))
    start = {"c": cast(grids["c"]), **{k: cast(adjs[k]) for k in ("c_b", "u_1_b", "u_2_b", "u_b")}}
    # the caller of the per-step ABI
    ref = {k: v.copy() for k, v in start.items()}
    plan = api.Plan(name, n, dtype)
    for u_1 in states:
        ref["u_1"] = u_1.copy()
        plan.run_adjoint_host(scalars, ref)
        ref["u_b"], ref["u_1_b"], ref["u_2_b"] = ref["u_1_b"], ref["u_2_b"], np.zeros_like(u_1)
    # the sweep
    host = {k: v.copy() for k, v in start.items()}
    plan.sweep_begin(host)
    for u_1 in states:
        plan.sweep_step_host(scalars, {"u_1": u_1})
    for k in ("c_b", "u_1_b", "u_2_b", "u_b"):
        host[k][...] = np.nan
    plan.sweep_end(host)
    plan.close()
    for k in ("c_b", "u_1_b", "u_2_b", "u_b"):
        assert np.array_equal(host[k], ref[k]), k
    assert not host["u_2_b"].any()


@pytest.mark.parametrize("n", [24, 40, 68, 97])
def test_plane_kernels_tma_equals_plain_fp64(api, n, sgbopt):
    """fp64 radius-4 plane kernels (the general-shape path behind the
    register-blocked kernel): the TMA-fed plane kernel (even n) and the
    plain-load plane kernel apply the same arithmetic per point (bitwise
    equal); both match the oracle at 1e-12.  Odd n takes the plain kernel."""
    name = "wave3d_r4"
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n + 9, accumulate=True)
    want = oracle_gather(name, n, scalars, grids, adjs)
    with sgbopt.context() as m:
        m.setenv("SGB_F64_PLANE", "1")
        base = api.run_program(name, n, scalars, grids, adjs, dtype="f64")
        m.setenv("SGB_PLANE_NO_TMA", "1")
        plain = api.run_program(name, n, scalars, grids, adjs, dtype="f64")
    for adj in ("c_b", "u_1_b"):
        check_close(base[adj], want[adj], "f64", f"n={n} {adj}")
        assert np.array_equal(plain[adj], base[adj]), adj


@pytest.mark.parametrize("name,n", [("wave3d_r4", n) for n in (20, 24, 40, 66, 98, 136)] +
                         [("wave3d_c", n) for n in (6, 16, 34, 66, 100)] +
                         [("wave3d_c2", n) for n in (12, 64)])
def test_f64_streaming_kernel(api, name, n, sgbopt):
    """fp64 register-blocked streaming kernel (even n; radius 4 and the
    radius-1 specs with their u_2 partial): matches the oracle at 1e-12 per
    point on the accumulated adjoints (partial tiles, frame tiles, one-tile
    grids); the i-chunk count changes only which CTA streams which planes
    (bitwise equal)."""
    scalars, grids, adjs = gen.family_inputs(name, n, seed=n + 21, accumulate=True)
    want = oracle_gather(name, n, scalars, grids, adjs)
    base = api.run_program(name, n, scalars, grids, adjs, dtype="f64")
    outs = [k for k in base if k != oracle.family(name).seed]
    for adj in outs:
        check_close(base[adj], want[adj], "f64", f"{name} n={n} {adj}")
    for chunks in ("1", "3", "7"):
        with sgbopt.context() as m:
            m.setenv("SGB_F64_ICHUNKS", chunks)
            got = api.run_program(name, n, scalars, grids, adjs, dtype="f64")
        for adj in outs:
            assert np.array_equal(got[adj], base[adj]), (chunks, adj)


@pytest.mark.parametrize("name,kind", [("wave3d_c", "adjoint"), ("wave3d_c", "fresh_u2"),
                                       ("wave3d_r4", "adjoint"), ("wave3d_r4", "fresh")])
def test_misaligned_arrays_take_a_safe_path(api, name, kind):
    """Arrays at a 4-byte offset (a contiguous view of a larger buffer, or an
    offset pointer from a C caller) cannot use the TMA / 16-byte vector
    kernels: the entry takes the per-point path instead of faulting, and the
    result still matches the aligned call."""
    import torch
    from paper_1907_02818_b200 import api as A
    n = 40
    sc = {"D": 0.1 if name == "wave3d_c" else 0.01}
    g = torch.Generator(device="cpu").manual_seed(5)
    names = A.array_params(name, "adjoint")
    aligned = {k: torch.randn((n, n, n), generator=g).cuda() for k in names}
    off = {}
    for k, v in aligned.items():
        buf = torch.empty(n ** 3 + 1, device="cuda")
        t = buf[1:].view(n, n, n)
        t.copy_(v)
        assert t.data_ptr() % 16 != 0
        off[k] = t
    call = {"adjoint": A.adjoint, "fresh_u2": A.adjoint_fresh_u2, "fresh": A.adjoint_fresh}[kind]
    call(name, n, sc, aligned)
    call(name, n, sc, off)
    torch.cuda.synchronize()
    for k in names:
        a, b = aligned[k].double().cpu().numpy(), off[k].double().cpu().numpy()
        assert oracle.max_rel_err(b, a) <= 1e-5, k
    # the context is healthy afterwards
    assert float(torch.ones(4, device="cuda").sum()) == 4.0
