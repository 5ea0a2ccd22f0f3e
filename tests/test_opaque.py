"""Opaque calls: an uninterpreted function f(a=.., b=..)
in the primal differentiates into named derivative calls f_d_a / f_d_b
(symdiff.cpp:277-288) that a back end maps to user code (PAPER §3.3.1).  The
reference renders them as C calls against declared prototypes
(codegen.cpp:153-168); the emitter renders them as calls to user-supplied
__device__ functions.  The interpreter cannot evaluate opaque calls
(interp.cpp:123-125), so the parity anchor is the reference's own emitted C,
compiled here with the same user functions written in C.

Problems come from `ref_harness ... opaque:<name>` (built through the
reference's expression builders; the JSON front end has no opaque syntax).
"""
import ctypes
import json
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle

needs_ref = pytest.mark.skipif(not oracle.ref_available(),
                               reason="oracle/_ref/ref_harness not built")

PROBLEMS = ["opaque:paper2d", "opaque:line1d"]

C_FUNCS = """
double f(double a, double b) { return a * a * b + 3.0 * b; }
double f_d_a(double a, double b) { return 2.0 * a * b; }
double f_d_b(double a, double b) { return a * a + 3.0; }
double g(double x, double y) { return x * y * y - x; }
double g_d_x(double x, double y) { return y * y - 1.0; }
double g_d_y(double x, double y) { return 2.0 * x * y; }
"""
CUDA_FUNCS = """
__device__ T f(T a, T b) { return a * a * b + T(3.0) * b; }
__device__ T f_d_a(T a, T b) { return T(2.0) * a * b; }
__device__ T f_d_b(T a, T b) { return a * a + T(3.0); }
__device__ T g(T x, T y) { return x * y * y - x; }
__device__ T g_d_x(T x, T y) { return y * y - T(1.0); }
__device__ T g_d_y(T x, T y) { return T(2.0) * x * y; }
"""


def harness(*args):
    r = subprocess.run([oracle.ref_harness_path(), *map(str, args)], capture_output=True,
                       text=True, timeout=300)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return r.stdout


class RefC:
    """The reference's emitted primal / gather adjoint for a problem, compiled
    with gcc together with the C user functions."""

    def __init__(self, problem, tmp):
        harness("emit", problem, tmp)
        self.spec = json.loads(harness("spec", problem))
        name = self.spec["name"]
        funcs = os.path.join(tmp, "funcs.c")
        with open(funcs, "w") as fh:
            fh.write(C_FUNCS)
        so = os.path.join(tmp, f"lib{name}.so")
        srcs = [os.path.join(tmp, f"{name}_primal.c"), os.path.join(tmp, f"{name}_adjoint.c")]
        subprocess.run(["/usr/bin/gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", so, *srcs,
                        funcs, "-lm"], check=True, capture_output=True)
        self.lib = ctypes.CDLL(so)
        self.sig = {}
        for which, src in (("primal", srcs[0]), ("adjoint", srcs[1])):
            text = open(src).read()
            fn = name + ("_b" if which == "adjoint" else "")
            m = re.search(rf"int {fn}\(([^)]*)\)", text)
            params = [p.strip() for p in m.group(1).split(",")]
            self.sig[which] = (fn, params)

    def call(self, which, sizes, scalars, arrays):
        fn, params = self.sig[which]
        args = []
        for p in params:
            name = p.split()[-1].lstrip("*")
            if p.startswith("int "):
                args.append(ctypes.c_int(int(sizes[name])))
            elif "*" in p:
                a = arrays[name]
                assert a.dtype == np.float64 and a.flags.c_contiguous
                args.append(a.ctypes.data_as(ctypes.c_void_p))
            else:
                args.append(ctypes.c_double(float(scalars[name])))
        return getattr(self.lib, fn)(*args)


def problem(name, n):
    spec = json.loads(harness("spec", name))
    info = json.loads(harness("info", name, n))
    return spec, info


def inputs(ep, n, seed):
    rng = np.random.default_rng(seed)
    out = {}
    for arr in ep.param_arrays("all"):
        shp = tuple(ep._eval_aff(a, {"n": n}) for a in ep._shape_of(arr))
        out[arr] = rng.standard_normal(shp)
    return out


def test_derivative_syntax_parses_to_opaque_calls():
    from paper_1907_02818_b200 import emitter
    e = emitter.parse_expr("c[i][j]*derivative(f, a)(a=u[i - 1][j], b=u[i][j - 1])")
    assert e[0] == "mul" and e[2][0] == "opaque" and e[2][1] == "f_d_a"
    assert [k for k, _ in e[2][2]] == ["a", "b"]
    call = emitter.parse_expr("f(a=u[i - 1][j], b=u[i][j - 1]) + 1")
    assert call[1] == ("opaque", "f", [("a", ("read", "u", [("i", -1), ("j", 0)])),
                                       ("b", ("read", "u", [("i", 0), ("j", -1)]))])
    with pytest.raises(ValueError):
        emitter.parse_expr("h(u[i])")  # positional opaque call: not the printed syntax


@needs_ref
@pytest.mark.parametrize("name", PROBLEMS)
def test_opaque_terms_and_emitted_kernels(name):
    """The front end's terms carry derivative calls; the emitted CUDA (with
    the user's device functions) compiles for sm_100a; its signature is the
    reference's."""
    from paper_1907_02818_b200 import emitter
    spec, info = problem(name, 12)
    assert any("derivative(" in t["partial"] for t in info["terms"])
    ep = emitter.EmittedProblem(spec, info["terms"], device_functions=CUDA_FUNCS)
    ep.check_compiles()
    assert "f_d_a(" in ep.gather_source() or "g_d_x(" in ep.gather_source()
    with tempfile.TemporaryDirectory() as td:
        ref = RefC(name, td)
    assert ep.param_arrays("gather") == [p.split()[-1].lstrip("*")
                                         for p in ref.sig["adjoint"][1] if "*" in p]
    assert ep.param_arrays("primal") == [p.split()[-1].lstrip("*")
                                         for p in ref.sig["primal"][1] if "*" in p]


@needs_ref
@pytest.mark.parametrize("name", PROBLEMS)
def test_reference_emitted_c_with_user_functions_passes_dot_test(name):
    """Fixture check (CPU): the C user derivatives are the derivatives of the
    C user functions -- the reference's emitted primal and adjoint satisfy
    <(F(u+hv) - F(u-hv)) / 2h, w> = <v, J^T w> (interp.cpp:300-381 method)."""
    from paper_1907_02818_b200 import emitter
    n = 24
    spec, info = problem(name, n)
    ep = emitter.EmittedProblem(spec, info["terms"])
    with tempfile.TemporaryDirectory() as td:
        ref = RefC(name, td)
        rng = np.random.default_rng(5)
        base = inputs(ep, n, 6)
        out, seed = ep.out, ep.seed
        active_in = [a for a, d in ep.arrays.items() if d["active"] and a != out]
        v = {a: rng.standard_normal(base[a].shape) for a in active_in}
        w = rng.standard_normal(base[out].shape)
        h = 1e-6
        sc = {"a": 0.7}

        def F(sign):
            arr = {k: x.copy() for k, x in base.items()}
            for a in active_in:
                arr[a] = arr[a] + sign * h * v[a]
            assert ref.call("primal", {"n": n}, sc, arr) == 0
            return arr[out]
        lhs = float(np.sum((F(1) - F(-1)) / (2 * h) * w))
        arr = {k: x.copy() for k, x in base.items()}
        for a in active_in:
            arr[ep.arrays[a]["adjoint"]] = np.zeros_like(base[a])
        arr[seed] = w.copy()
        assert ref.call("adjoint", {"n": n}, sc, arr) == 0
        rhs = float(sum(np.sum(v[a] * arr[ep.arrays[a]["adjoint"]]) for a in active_in))
    assert abs(lhs - rhs) <= 1e-6 * max(1.0, abs(rhs)), (lhs, rhs)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("name", PROBLEMS)
@pytest.mark.parametrize("n", [12, 37])
def test_opaque_emitted_kernels_match_reference_emitted_c(name, n):
    """GPU parity: gather adjoint and primal of the emitted CUDA (user device
    functions) against the reference's emitted C (same functions in C), fp64,
    compare_grids <= 1e-12; the per-nest form equals the fused form bitwise."""
    import torch
    from paper_1907_02818_b200 import emitter
    spec, info = problem(name, n)
    ep = emitter.EmittedProblem(spec, info["terms"], device_functions=CUDA_FUNCS)
    sc = {"a": 0.37}
    host = inputs(ep, n, n)
    with tempfile.TemporaryDirectory() as td:
        ref = RefC(name, td)
        want = {k: v.copy() for k, v in host.items()}
        assert ref.call("adjoint", {"n": n}, sc, want) == 0
        want_p = {k: v.copy() for k, v in host.items()}
        assert ref.call("primal", {"n": n}, sc, want_p) == 0
    dev = {k: torch.from_numpy(v.copy()).cuda() for k, v in host.items()}
    ep.adjoint({"n": n}, sc, dev)
    nest = {k: torch.from_numpy(v.copy()).cuda() for k, v in host.items()}
    ep.adjoint_nests({"n": n}, sc, nest)
    prim = {k: torch.from_numpy(v.copy()).cuda() for k, v in host.items()}
    ep.primal({"n": n}, sc, prim)
    torch.cuda.synchronize()
    for t in {t["adjoint"] for t in info["terms"]}:
        got = dev[t].cpu().numpy()
        assert oracle.max_rel_err(got, want[t]) <= 1e-12, (name, t)
        assert torch.equal(dev[t], nest[t]), (name, t)
    assert oracle.max_rel_err(prim[ep.out].cpu().numpy(), want_p[ep.out]) <= 1e-12
