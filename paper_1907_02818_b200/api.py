"""Host-side API over the C ABI (include/stencilgrad_b200.h).

Two layers, mirroring the reference's two interfaces:

* generated-function layer on DEVICE tensors -- ``primal`` / ``adjoint`` /
  ``scatter_adjoint`` call ``<name>``, ``<name>_b``, ``<name>_scatter_b``
  (codegen.cpp:311-434) with arguments gathered by parameter name from a dict
  of torch CUDA tensors, on the current torch stream;
* in-memory layer on HOST numpy grids -- ``run_nest`` / ``run_program`` /
  ``run_scatter_adjoint`` take ``(family, n, scalars, grids, adjoints)`` and
  return new arrays, leaving the inputs untouched, like the reference's
  ``Env run_program(const AdjointProgram&, const Env&)`` (interp.hpp:56-63).
  They upload, run the sm_100a kernels and download.

Unsupported families, shapes or dtypes raise; there is no CPU fallback.
torch is only the device-memory / stream plumbing here.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

FAMILIES = {"wave1d": 1, "wave3d_c": 3, "wave3d_c2": 3, "burgers2d": 2, "wave3d_r4": 3}
SCALARS = {"wave1d": ["D"], "wave3d_c": ["D"], "wave3d_c2": ["D"], "burgers2d": ["C", "D"],
           "wave3d_r4": ["D"]}
_SUFFIX = {"primal": "", "adjoint": "_b", "scatter": "_scatter_b", "slab": "_b_slab",
           "fresh": "_b_fresh", "fresh_slab": "_b_fresh_slab", "fresh_u2": "_b_fresh_u2"}


def _sfx(dtype) -> str:
    import torch
    if dtype in (torch.float32, np.float32, "f32", "float32"):
        return "f32"
    if dtype in (torch.float64, np.float64, "f64", "float64"):
        return "f64"
    raise _lib.StencilError(f"unsupported dtype {dtype} (f32 or f64 only)")


def function_name(family: str, kind: str, dtype) -> str:
    if family not in FAMILIES:
        raise _lib.StencilError(f"unsupported stencil family '{family}'")
    if kind not in _SUFFIX:
        raise _lib.StencilError(f"unknown entry kind '{kind}'")
    name = f"{family}{_SUFFIX[kind]}_{_sfx(dtype)}"
    if name not in _lib.PROTOTYPES:
        raise _lib.StencilError(f"no entry point {name} in stencilgrad_b200.h "
                                f"('{kind}' is not provided for {family} in this precision)")
    return name


def array_params(family: str, kind: str, dtype="f32"):
    """Array parameter names of the C entry point, in prototype order."""
    _, params = _lib.PROTOTYPES[function_name(family, kind, dtype)]
    return [p for t, p in params if t.endswith("*") and t not in ("const char*",)]


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _call(family, kind, n, scalars, arrays, stream=None, extra=()):
    names = array_params(family, kind)
    d = FAMILIES[family]
    # every array holds the full n^d grid (a slab: nplanes whole planes); a
    # short buffer would be read out of bounds, so it is rejected here like
    # the reference's bounds error (interp.cpp:30-35)
    want = int(extra[1]) * int(n) ** (d - 1) if kind.endswith("slab") else int(n) ** d
    dtype = None
    ptrs = []
    for nm in names:
        t = arrays.get(nm)
        if t is None:
            raise _lib.StencilError(f"{family}{_SUFFIX[kind]}: missing array '{nm}'")
        if not (t.is_cuda and t.is_contiguous()):
            raise _lib.StencilError(f"array '{nm}' must be a contiguous CUDA tensor")
        if t.numel() != want:
            raise _lib.StencilError(f"array '{nm}' has {t.numel()} elements, expected {want}")
        if dtype is None:
            dtype = t.dtype
        elif t.dtype != dtype:
            raise _lib.StencilError("all arrays must share one dtype")
        ptrs.append(ctypes.c_void_p(t.data_ptr()))
    fname = function_name(family, kind, dtype)
    fn = getattr(_lib.lib(), fname)
    sc = [float(scalars[s]) for s in SCALARS[family]]
    rc = fn(int(n), *sc, *ptrs, *extra, _stream_ptr(stream))
    _lib.check(rc, fname)


def primal(family, n, scalars, arrays, stream=None):
    """<name>_{f32,f64}: primal stencil (run_nest semantics, interp.cpp:153-173)."""
    _call(family, "primal", n, scalars, arrays, stream)


def adjoint(family, n, scalars, arrays, stream=None):
    """<name>_b_{f32,f64}: fused core+boundary gather adjoint, accumulating (+=)."""
    _call(family, "adjoint", n, scalars, arrays, stream)


def scatter_adjoint(family, n, scalars, arrays, stream=None):
    """<name>_scatter_b_{f32,f64}: atomic scatter adjoint (ablation)."""
    _call(family, "scatter", n, scalars, arrays, stream)


def adjoint_slab(family, n, scalars, arrays, i_base, nplanes, out_i0, out_i1, stream=None):
    """z-slab gather adjoint over global output planes [out_i0, out_i1)."""
    _call(family, "slab", n, scalars, arrays, stream,
          extra=(int(i_base), int(nplanes), int(out_i0), int(out_i1)))


def adjoint_fresh(family, n, scalars, arrays, stream=None):
    """wave3d_r4_b_fresh_f32: the gather adjoint with u_1_b = this call's
    adjoint alone (c_b accumulated) -- zeroing u_1_b and accumulating, fused."""
    _call(family, "fresh", n, scalars, arrays, stream)


def adjoint_slab_fresh(family, n, scalars, arrays, i_base, nplanes, out_i0, out_i1,
                       stream=None):
    """z-slab form of adjoint_fresh over global output planes [out_i0, out_i1)."""
    _call(family, "fresh_slab", n, scalars, arrays, stream,
          extra=(int(i_base), int(nplanes), int(out_i0), int(out_i1)))


def adjoint_fresh_u2(family, n, scalars, arrays, stream=None):
    """wave3d_c(2)_b_fresh_u2_f32: the radius-1 gather with u_2_b = this call's
    u_2 partial alone (a carried sweep's zeroing of u_2_b, fused)."""
    _call(family, "fresh_u2", n, scalars, arrays, stream)


# ------------------------------------------------------------ device inputs
def fill_random(t, index_base: int, seed: int, stream_id: int, kind: str, a: float, b: float,
                stream=None):
    """kind 'normal': N(a, b^2); 'uniform': U[a, a + b). Counter-based in the
    GLOBAL flat index, so any slab regenerates the single-GPU values."""
    import torch
    k = {"normal": 0, "uniform": 1}[kind]
    fn = _lib.lib().sgb_fill_random_f32 if t.dtype == torch.float32 else \
        _lib.lib().sgb_fill_random_f64
    _lib.check(fn(ctypes.c_void_p(t.data_ptr()), t.numel(), int(index_base), int(seed),
                  int(stream_id), k, float(a), float(b), _stream_ptr(stream)), "fill_random")


def fill_normal3d(t, n: int, halo: int, seed: int, stream_id: int, i_base: int = 0,
                  nplanes: int | None = None, mean: float = 0.0, scale: float = 1.0,
                  stream=None):
    """N(mean, scale^2) on planes [i_base, i_base+nplanes) of an n^3 grid
    with a zero `halo`-point shell, in one pass (same values as fill_random;
    an fp64 tensor gets the fp32 values widened)."""
    import torch
    fn = _lib.lib().sgb_fill_normal3d_f32 if t.dtype == torch.float32 else \
        _lib.lib().sgb_fill_normal3d_f64
    _lib.check(fn(ctypes.c_void_p(t.data_ptr()), n, i_base, n if nplanes is None else nplanes,
                  halo, int(seed), int(stream_id), float(mean), float(scale),
                  _stream_ptr(stream)), "fill_normal3d")


def fill_normal3d_pair(a, halo_a: int, stream_a: int, b, halo_b: int, stream_b: int, n: int,
                       seed: int, i_base: int = 0, nplanes: int | None = None,
                       mean: float = 0.0, scale: float = 1.0, stream=None):
    """Two fields in one pass: bitwise fill_normal3d(a, n, halo_a, seed,
    stream_a, ...) and fill_normal3d(b, n, halo_b, seed, stream_b, ...)."""
    import torch
    if a.dtype != b.dtype:
        raise _lib.StencilError("fill_normal3d_pair: both fields must share one dtype")
    fn = _lib.lib().sgb_fill_normal3d_pair_f32 if a.dtype == torch.float32 else \
        _lib.lib().sgb_fill_normal3d_pair_f64
    _lib.check(fn(ctypes.c_void_p(a.data_ptr()), int(halo_a), int(stream_a),
                  ctypes.c_void_p(b.data_ptr()), int(halo_b), int(stream_b), n, i_base,
                  n if nplanes is None else nplanes, int(seed), float(mean), float(scale),
                  _stream_ptr(stream)), "fill_normal3d_pair")


def zero_halo(t, d: int, n: int, h: int, i_base: int = 0, nplanes: int | None = None,
              stream=None):
    import torch
    fn = _lib.lib().sgb_zero_halo_f32 if t.dtype == torch.float32 else _lib.lib().sgb_zero_halo_f64
    _lib.check(fn(ctypes.c_void_p(t.data_ptr()), d, n, h, i_base,
                  n if nplanes is None else nplanes, _stream_ptr(stream)), "zero_halo")


def fill_layered(t, n: int, layers: int, lo: float, hi: float, seed: int, i_base: int = 0,
                 nplanes: int | None = None, stream=None):
    _lib.check(_lib.lib().sgb_fill_layered_f32(
        ctypes.c_void_p(t.data_ptr()), n, layers, lo, hi, seed, i_base,
        n if nplanes is None else nplanes, _stream_ptr(stream)), "fill_layered")


def box_axpy(y, x, alpha: float, n: int, lo: int, hi: int, i_base: int = 0,
             nplanes: int | None = None, stream=None):
    """y[B] += alpha * x[B] for the box B = [lo, hi]^3 (3D grids)."""
    import torch
    fn = _lib.lib().sgb_box_axpy_f32 if y.dtype == torch.float32 else _lib.lib().sgb_box_axpy_f64
    _lib.check(fn(ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(x.data_ptr()), float(alpha), n,
                  lo, hi, i_base, n if nplanes is None else nplanes, _stream_ptr(stream)),
               "box_axpy")


def box_set(y, x, alpha: float, n: int, lo: int, hi: int, i_base: int = 0,
            nplanes: int | None = None, stream=None):
    """y = alpha * x on the box B = [lo, hi]^3, 0 elsewhere (3D grids)."""
    import torch
    fn = _lib.lib().sgb_box_set_f32 if y.dtype == torch.float32 else _lib.lib().sgb_box_set_f64
    _lib.check(fn(ctypes.c_void_p(y.data_ptr()), ctypes.c_void_p(x.data_ptr()), float(alpha), n,
                  lo, hi, i_base, n if nplanes is None else nplanes, _stream_ptr(stream)),
               "box_set")


def adjoint_time_step(n: int, scalars, arrays, u_2_b, stream=None):
    """One reverse step of a wave3d_r4 time loop (fp32, device arrays): the
    gather adjoint (c_b, u_1_b accumulated from the seed u_b) and the u_2
    partial u_2_b = -u_b on [4, n-5]^3, 0 elsewhere, fused into the gather
    kernel (sgb_wave3d_r4_b_step_f32)."""
    import torch
    names = array_params("wave3d_r4", "adjoint")
    ts = [arrays.get(k) for k in names] + [u_2_b]
    for nm, t in zip(names + ["u_2_b"], ts):
        if t is None or not (t.is_cuda and t.is_contiguous()) or t.dtype != torch.float32 \
                or t.numel() != int(n) ** 3:
            raise _lib.StencilError(f"adjoint_time_step: '{nm}' must be a contiguous fp32 "
                                    f"CUDA tensor of {n}^3 elements")
    ptr = [ctypes.c_void_p(t.data_ptr()) for t in ts[:-1]]
    _lib.check(_lib.lib().sgb_wave3d_r4_b_step_f32(
        n, float(scalars["D"]), *ptr, ctypes.c_void_p(u_2_b.data_ptr()), _stream_ptr(stream)),
        "sgb_wave3d_r4_b_step_f32")


def smooth5(src, dst, n: int, stream=None):
    _lib.check(_lib.lib().sgb_smooth5_f64(ctypes.c_void_p(src.data_ptr()),
                                          ctypes.c_void_p(dst.data_ptr()), n,
                                          _stream_ptr(stream)), "smooth5")


# ------------------------------------------------------------ host (Env-style) layer
def _to_dev(a: np.ndarray, dtype):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


def _run_host(kind, family, n, scalars, grids, adjs, dtype):
    import torch
    td = torch.float32 if _sfx(dtype) == "f32" else torch.float64
    arrays = {}
    for k, v in {**grids, **adjs}.items():
        arrays[k] = _to_dev(v, td)
    _call(family, kind, n, scalars, arrays)
    torch.cuda.synchronize()
    return {k: arrays[k].to("cpu", torch.float64).numpy() for k in arrays}


def run_nest(family, n, scalars, grids, dtype="f64"):
    """Primal on the B200; returns a new dict of host grids (interp.hpp:56)."""
    return _run_host("primal", family, n, scalars, grids, {}, dtype)


def run_program(family, n, scalars, grids, adjs, dtype="f64"):
    """Gather adjoint on the B200; returns new host arrays (interp.hpp:59)."""
    out = _run_host("adjoint", family, n, scalars, grids, adjs, dtype)
    return {k: out[k] for k in adjs}


def run_scatter_adjoint(family, n, scalars, grids, adjs, dtype="f64"):
    """Atomic scatter adjoint on the B200 (interp.hpp:63)."""
    out = _run_host("scatter", family, n, scalars, grids, adjs, dtype)
    return {k: out[k] for k in adjs}


class Plan:
    """Device workspace for the host-buffer entry point (sgb_plan_*)."""

    def __init__(self, family: str, n: int, dtype="f32", slab=None):
        """slab: a slab.Slab (multi-GPU host-buffer path: host arrays hold the
        local planes, outputs are the owned planes); None = the full grid."""
        self.family, self.n = family, n
        self.dtype_bytes = 4 if _sfx(dtype) == "f32" else 8
        if slab is None:
            self._p = _lib.lib().sgb_plan_create(family.encode(), n, self.dtype_bytes)
        else:
            self._p = _lib.lib().sgb_plan_create_slab(family.encode(), n, self.dtype_bytes,
                                                      slab.base, slab.nplanes, slab.own0,
                                                      slab.own1)
        if not self._p:
            raise _lib.StencilError(_lib.lib().sgb_last_error().decode())
        self.names = array_params(family, "adjoint")

    def run_adjoint_host(self, scalars: dict, host_arrays: dict, stream=None):
        """host_arrays: name -> pinned CPU tensor or numpy array (dtype of the plan)."""
        ptrs = (ctypes.c_void_p * len(self.names))()
        for i, nm in enumerate(self.names):
            a = host_arrays[nm]
            ptrs[i] = a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        sc = (ctypes.c_double * 2)(*[float(scalars[s]) for s in SCALARS[self.family]])
        s = ctypes.c_void_p(0) if stream is None else _stream_ptr(stream)
        _lib.check(_lib.lib().sgb_plan_run_adjoint_host(ctypes.c_void_p(self._p), sc, ptrs, s),
                   "sgb_plan_run_adjoint_host")

    def _ptrs(self, host_arrays: dict, needed):
        ptrs = (ctypes.c_void_p * len(self.names))()
        for i, nm in enumerate(self.names):
            a = host_arrays.get(nm)
            if a is None:
                if nm in needed:
                    raise _lib.StencilError(f"Plan: host array {nm} missing")
                continue
            ptrs[i] = a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data
        return ptrs

    # sgb_plan_sweep_*: which host arrays each call touches, per family
    _SWEEP = {"wave3d_r4": (("c", "c_b"), ("u_1", "u_1_b", "u_b"), ("c_b",)),
              "wave3d_c": (("c", "c_b", "u_1_b", "u_2_b", "u_b"), ("u_1",),
                           ("c_b", "u_1_b", "u_2_b", "u_b"))}

    def _sweep_names(self, i):
        return self._SWEEP.get(self.family, ((), (), ()))[i]

    def sweep_begin(self, host_arrays: dict, stream=None):
        """Start a reverse sweep over host-held states (sgb_plan_sweep_*): what
        does not change per step goes to the device once and stays there
        (wave3d_r4: c, c_b; wave3d_c: c, c_b and the carried adjoints)."""
        s = ctypes.c_void_p(0) if stream is None else _stream_ptr(stream)
        _lib.check(_lib.lib().sgb_plan_sweep_begin(
            ctypes.c_void_p(self._p), self._ptrs(host_arrays, self._sweep_names(0)), s),
            "sgb_plan_sweep_begin")

    def sweep_step_host(self, scalars: dict, host_arrays: dict, stream=None):
        """One reverse step.  wave3d_r4: u_1, u_b in, u_1_b (this step's adjoint
        alone) out, c_b accumulates on the device.  wave3d_c: u_1 in; the
        adjoints accumulate and rotate on the device."""
        sc = (ctypes.c_double * 2)(*[float(scalars[s]) for s in SCALARS[self.family]])
        s = ctypes.c_void_p(0) if stream is None else _stream_ptr(stream)
        _lib.check(_lib.lib().sgb_plan_sweep_step_host(
            ctypes.c_void_p(self._p), sc, self._ptrs(host_arrays, self._sweep_names(1)), s),
            "sgb_plan_sweep_step_host")

    def sweep_end(self, host_arrays: dict, stream=None):
        """Finish the sweep: the device-resident results come back to the host."""
        s = ctypes.c_void_p(0) if stream is None else _stream_ptr(stream)
        _lib.check(_lib.lib().sgb_plan_sweep_end(
            ctypes.c_void_p(self._p), self._ptrs(host_arrays, self._sweep_names(2)), s),
            "sgb_plan_sweep_end")

    def close(self):
        if self._p:
            _lib.lib().sgb_plan_destroy(ctypes.c_void_p(self._p))
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------ device parity reductions
def compare(a, b):
    """compare_grids (interp.cpp:290-298) on the device: a (fp32 / fp64 CUDA
    tensor) against the fp64 CUDA tensor b.  Returns {"max_rel": max |a-b| /
    (1+|b|), "norm_rel": ||a-b|| / ||b||, "nonfinite": count}."""
    import math
    import torch
    if not (a.is_cuda and b.is_cuda and a.is_contiguous() and b.is_contiguous()):
        raise _lib.StencilError("compare: contiguous CUDA tensors required")
    if b.dtype != torch.float64 or a.numel() != b.numel():
        raise _lib.StencilError("compare: b must be fp64 with a's element count")
    fn = {torch.float32: _lib.lib().sgb_compare_f32,
          torch.float64: _lib.lib().sgb_compare_f64}.get(a.dtype)
    if fn is None:
        raise _lib.StencilError(f"compare: unsupported dtype {a.dtype}")
    out = (ctypes.c_double * 4)()
    _lib.check(fn(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()), a.numel(), out,
                  _stream_ptr()), "compare")
    nb = math.sqrt(out[2])
    return {"max_rel": out[0], "norm_rel": math.sqrt(out[1]) / (nb if nb > 0 else 1.0),
            "nonfinite": int(out[3])}


def dot(a, b):
    """<a, b> accumulated in fp64 on the device (dot_product_test's inner
    products, interp.cpp:354-375)."""
    import torch
    if a.dtype != b.dtype or a.numel() != b.numel() or not (a.is_cuda and b.is_cuda):
        raise _lib.StencilError("dot: CUDA tensors of one dtype and size required")
    fn = {torch.float32: _lib.lib().sgb_dot_f32, torch.float64: _lib.lib().sgb_dot_f64}.get(
        a.dtype)
    if fn is None:
        raise _lib.StencilError(f"dot: unsupported dtype {a.dtype}")
    out = ctypes.c_double()
    _lib.check(fn(ctypes.c_void_p(a.contiguous().data_ptr()),
                  ctypes.c_void_p(b.contiguous().data_ptr()), a.numel(), ctypes.byref(out),
                  _stream_ptr()), "dot")
    return out.value


# ------------------------------------------------------------ run-time options
def option_names():
    out, i = [], 0
    while True:
        nm = _lib.lib().sgb_option_name(i)
        if nm is None:
            return out
        out.append(nm.decode())
        i += 1


def get_option(name: str):
    """(value, is_set) of a run-time option (sgb_get_option)."""
    v, s = ctypes.c_longlong(), ctypes.c_int()
    _lib.check(_lib.lib().sgb_get_option(name.encode(), ctypes.byref(v), ctypes.byref(s)),
               "sgb_get_option")
    return v.value, bool(s.value)


def set_option(name: str, value=None):
    """Sets (value not None) or clears a run-time option (sgb_set_option)."""
    L = _lib.lib()
    if value is None:
        _lib.check(L.sgb_clear_option(name.encode()), "sgb_clear_option")
    else:
        _lib.check(L.sgb_set_option(name.encode(), int(value)), "sgb_set_option")


class options:
    """Context manager: ``with api.options(NO_UBWIN=1, ICHUNKS=3): ...``
    restores the previous settings on exit."""

    def __init__(self, **kw):
        self.kw = kw
        self.saved = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.saved[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, (v, was_set) in self.saved.items():
            set_option(k, v if was_set else None)


# ------------------------------------------------------------ program-keyed entry
_PROG_DIR = __import__("os").path.join(__import__("os").path.dirname(
    __import__("os").path.abspath(__file__)), "programs")


def load_program(name: str) -> dict:
    """A reference front-end output committed under programs/<name>.json:
    {"spec": serialize_spec (specfile.cpp:208-240), "terms": the
    AdjointProgram's terms in active_reads order with to_input_string
    partials (adjoint.hpp:13-19)}."""
    import json
    import os
    with open(os.path.join(_PROG_DIR, name + ".json")) as fh:
        d = json.load(fh)
    return {"spec": d["spec"], "terms": d["terms"]}


def _norm_program(p: dict):
    import json
    terms = [{"array": t["array"], "adjoint": t["adjoint"], "offset": list(t["offset"]),
              "partial": " ".join(str(t["partial"]).split())} for t in p["terms"]]
    return json.dumps(p["spec"], sort_keys=True), json.dumps(terms)


def program_family(program: dict):
    """The family whose hand-tuned kernels compute exactly `program` (same
    spec -- counters, bounds, arrays, lhs, mode, rhs -- and the same terms:
    arrays, offsets, partials), or None."""
    key = _norm_program(program)
    for fam in FAMILIES:
        if _norm_program(load_program(fam)) == key:
            return fam
    return None


def run_program_from(program: dict, sizes: dict, scalars: dict, grids: dict, adjs: dict,
                     dtype="f64", return_route=False):
    """run_program(const AdjointProgram&, const Env&) (interp.hpp:59) keyed on
    the PROGRAM: a program one of the hand-tuned families computes runs those
    kernels; any other program is lowered through the NVRTC emitter
    (emitter.py), which consumes its terms and bounds.  Host grids in, new
    host adjoint arrays out (the inputs are untouched)."""
    fam = program_family(program)
    if fam is not None:
        out = run_program(fam, int(sizes["n"]), scalars, grids, adjs, dtype=dtype)
        return (out, "hand-tuned") if return_route else out
    import torch
    from . import emitter
    ep = emitter.EmittedProblem(program["spec"], program["terms"], _sfx(dtype))
    td = torch.float32 if _sfx(dtype) == "f32" else torch.float64
    arrays = {k: _to_dev(v, td) for k, v in {**grids, **adjs}.items()}
    ep.adjoint(sizes, scalars, arrays)
    torch.cuda.synchronize()
    out = {k: arrays[k].to("cpu", torch.float64).numpy() for k in adjs}
    return (out, "emitter") if return_route else out
