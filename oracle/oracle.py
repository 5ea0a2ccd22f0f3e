"""ctypes view of the CPU oracle (oracle/sg_oracle.c) and the reference harness.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs -- as the checker or the
timed CPU baseline, never as the product path.  The product package
(``paper_1907_02818_b200``) does not import this module.

Grids are numpy float64 arrays, row-major with the innermost counter contiguous
(interp.cpp:30-35).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")
SPEC_DIR = os.path.join(HERE, "specs")

MAX_TERMS = 32
MAX_ARRAYS = 6
MAX_NESTS = 4096

FAMILIES = ["wave1d", "wave3d_c", "wave3d_c2", "burgers2d", "wave3d_r4", "lap1d", "wave3d",
            "burgers1d"]


class _Family(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char_p), ("d", ctypes.c_int), ("lo", ctypes.c_int),
        ("hi_n", ctypes.c_int), ("shape_n", ctypes.c_int), ("nscalars", ctypes.c_int),
        ("scalars", ctypes.c_char_p * 2), ("narrays", ctypes.c_int),
        ("arrays", ctypes.c_char_p * MAX_ARRAYS), ("adjoints", ctypes.c_char_p * MAX_ARRAYS),
        ("output", ctypes.c_int), ("increment", ctypes.c_int), ("nterms", ctypes.c_int),
        ("term_array", ctypes.c_int * MAX_TERMS), ("term_off", (ctypes.c_int * 3) * MAX_TERMS),
        ("radius", ctypes.c_int),
    ]


class _Env(ctypes.Structure):
    _fields_ = [("n", ctypes.c_longlong), ("scalars", ctypes.c_double * 2),
                ("grid", ctypes.c_void_p * MAX_ARRAYS), ("adj", ctypes.c_void_p * MAX_ARRAYS)]


class _Nest(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_longlong * 3), ("hi", ctypes.c_longlong * 3),
                ("nterms", ctypes.c_int), ("terms", ctypes.c_int * MAX_TERMS),
                ("core", ctypes.c_int)]


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.sg_family_get.restype = ctypes.POINTER(_Family)
        L.sg_family_by_name.argtypes = [ctypes.c_char_p]
        L.sg_split_offsets.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.sg_split_family.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p,
                                      ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
        L.sg_core_bounds.argtypes = [ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p,
                                     ctypes.c_void_p]
        L.sg_check_guards.argtypes = [ctypes.c_int, ctypes.c_longlong]
        L.sg_array_len.argtypes = [ctypes.c_int, ctypes.c_longlong]
        L.sg_array_len.restype = ctypes.c_longlong
        for fn in ("sg_run_primal", "sg_run_program", "sg_run_program_predicate",
                   "sg_run_scatter", "sg_run_program_omp"):
            getattr(L, fn).argtypes = [ctypes.c_int, ctypes.POINTER(_Env)]
        L.sg_max_rel_err.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong]
        L.sg_max_rel_err.restype = ctypes.c_double
        _lib = L
    return _lib


@dataclass
class Family:
    id: int
    name: str
    d: int
    lo: int
    hi_n: int
    shape_n: int
    scalars: list
    arrays: list
    adjoints: list
    output: int
    increment: bool
    terms: list  # [(array_index, (o0, o1, o2)[:d])]
    radius: int

    def shape(self, n):
        return (n + self.shape_n,) * self.d

    def bounds(self, n):
        return [(self.lo, n + self.hi_n)] * self.d

    @property
    def seed(self):
        return self.adjoints[self.output]

    @property
    def active_inputs(self):
        """Active non-output arrays, declaration order (interp.cpp:309-311)."""
        return [a for i, a in enumerate(self.arrays) if self.adjoints[i] and i != self.output]


def family(name: str) -> Family:
    L = lib()
    fid = L.sg_family_by_name(name.encode())
    if fid < 0:
        raise KeyError(name)
    f = L.sg_family_get(fid).contents
    return Family(
        id=fid, name=f.name.decode(), d=f.d, lo=f.lo, hi_n=f.hi_n, shape_n=f.shape_n,
        scalars=[f.scalars[i].decode() for i in range(f.nscalars)],
        arrays=[f.arrays[i].decode() for i in range(f.narrays)],
        adjoints=[f.adjoints[i].decode() for i in range(f.narrays)],
        output=f.output, increment=bool(f.increment),
        terms=[(f.term_array[t], tuple(f.term_off[t][i] for i in range(f.d)))
               for t in range(f.nterms)],
        radius=f.radius)


def _nests_from(buf, count, d):
    out = []
    for k in range(count):
        ns = buf[k]
        out.append({"bounds": [(ns.lo[i], ns.hi[i]) for i in range(d)],
                    "terms": [ns.terms[a] for a in range(ns.nterms)], "core": bool(ns.core)})
    return out


def split_offsets(offsets, lo, hi):
    """Restated Splitter::recurse on explicit offsets (adjoint.cpp:73-150)."""
    d = len(offsets[0])
    off = ((ctypes.c_int * 3) * MAX_TERMS)()
    for t, o in enumerate(offsets):
        for i in range(d):
            off[t][i] = o[i]
    clo = (ctypes.c_longlong * 3)(*lo, *([0] * (3 - d)))
    chi = (ctypes.c_longlong * 3)(*hi, *([0] * (3 - d)))
    buf = (_Nest * MAX_NESTS)()
    core = ctypes.c_int(-1)
    cnt = lib().sg_split_offsets(d, len(offsets), off, clo, chi, buf, MAX_NESTS,
                                 ctypes.byref(core))
    if cnt < 0:
        raise ValueError("split overflow")
    return _nests_from(buf, cnt, d), core.value


def split_family(name: str, n: int):
    f = family(name)
    buf = (_Nest * MAX_NESTS)()
    core = ctypes.c_int(-1)
    cnt = lib().sg_split_family(f.id, n, buf, MAX_NESTS, ctypes.byref(core))
    if cnt < 0:
        raise ValueError("split overflow")
    return _nests_from(buf, cnt, f.d), core.value


def core_bounds(name: str, n: int):
    f = family(name)
    lo = (ctypes.c_longlong * 3)()
    hi = (ctypes.c_longlong * 3)()
    lib().sg_core_bounds(f.id, n, lo, hi)
    return [(lo[i], hi[i]) for i in range(f.d)]


def guards_ok(name: str, n: int) -> bool:
    return lib().sg_check_guards(family(name).id, n) == 0


def _env(f: Family, n: int, scalars: dict, grids: dict, adjs: dict):
    env = _Env()
    env.n = n
    for i, s in enumerate(f.scalars):
        env.scalars[i] = float(scalars[s])
    keep = []
    shape = f.shape(n)
    for i, a in enumerate(f.arrays):
        g = grids.get(a)
        if g is None:
            g = np.zeros(shape)
            grids[a] = g
        assert g.dtype == np.float64 and g.flags.c_contiguous and g.shape == shape, a
        env.grid[i] = g.ctypes.data
        keep.append(g)
        if f.adjoints[i]:
            b = adjs.get(f.adjoints[i])
            if b is None:
                b = np.zeros(shape)
                adjs[f.adjoints[i]] = b
            assert b.dtype == np.float64 and b.flags.c_contiguous and b.shape == shape
            env.adj[i] = b.ctypes.data
            keep.append(b)
    return env, keep


def _run(fn: str, name: str, n: int, scalars: dict, grids: dict, adjs: dict) -> int:
    f = family(name)
    env, _keep = _env(f, n, scalars, grids, adjs)
    return getattr(lib(), fn)(f.id, ctypes.byref(env))


def run_primal(name, n, scalars, grids, adjs=None):
    """run_nest restated; writes grids[output] in place."""
    return _run("sg_run_primal", name, n, scalars, grids, adjs if adjs is not None else {})


def run_program(name, n, scalars, grids, adjs):
    """run_program restated (hierarchical nests); accumulates into adjs in place."""
    return _run("sg_run_program", name, n, scalars, grids, adjs)


def run_program_predicate(name, n, scalars, grids, adjs):
    return _run("sg_run_program_predicate", name, n, scalars, grids, adjs)


def run_program_omp(name, n, scalars, grids, adjs):
    """OpenMP predicate form; returns the number of threads used (>= 1), or
    -1 on a guard violation."""
    return _run("sg_run_program_omp", name, n, scalars, grids, adjs)


def run_scatter(name, n, scalars, grids, adjs):
    return _run("sg_run_scatter", name, n, scalars, grids, adjs)


def max_rel_err(a: np.ndarray, b: np.ndarray) -> float:
    """compare_grids metric (interp.cpp:290-298)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape
    return float(lib().sg_max_rel_err(a.ctypes.data, b.ctypes.data, a.size))


def norm_rel_err(a: np.ndarray, b: np.ndarray) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = float(np.linalg.norm(b.ravel()))
    return float(np.linalg.norm((a - b).ravel())) / (nb if nb > 0 else 1.0)


# ---------------------------------------------------------------- reference harness
def ref_harness_path() -> str:
    return os.path.join(REF_DIR, "ref_harness")


def ref_available() -> bool:
    return os.path.exists(ref_harness_path())


def spec_path(name: str) -> str:
    p = os.path.join(SPEC_DIR, name + ".json")
    return p if os.path.exists(p) else "example:" + name


# ---------------------------------------------------------------- reference emitted C
def ref_emitted_path(name: str) -> str:
    return os.path.join(REF_DIR, f"libref_{name}.so")


def ref_emitted_available(name: str) -> bool:
    return os.path.exists(ref_emitted_path(name))


def ref_emitted_opt(name: str) -> str:
    p = os.path.join(REF_DIR, f"libref_{name}.opt")
    return open(p).read().strip() if os.path.exists(p) else "-O2"


def _ref_params(name: str, fn: str):
    """Parameter names of <fn> from the prototypes the reference emitted
    itself (oracle/_ref/gen/<name>_protos.h; codegen.cpp:198-230)."""
    import re
    text = open(os.path.join(REF_DIR, "gen", f"{name}_protos.h")).read()
    m = re.search(r"int\s+" + re.escape(fn) + r"\(([^)]*)\);", text)
    if not m:
        raise KeyError(fn)
    out = []
    for a in m.group(1).split(","):
        a = a.strip()
        out.append(("ptr" if "*" in a else a.split()[0], a.replace("*", " ").split()[-1]))
    return out


_ref_libs = {}


def emitted_or_port(name: str):
    """(call, label): the reference's own compiled emitted adjoint when
    oracle/_ref holds it (ref_emitted), else the pinned C restatement's OpenMP
    run_program (sg_run_program_omp, pinned to the reference's outputs by
    tests/test_oracle_pins.py) behind the same call(n, scalars, arrays)
    interface.  The radius-4 emitted adjoint is a ~12 min build (make -C
    oracle/ref ref_r4), so a fresh build container may lack it; parity is then
    anchored on the port, and the label says which oracle ran."""
    if ref_emitted_available(name):
        return ref_emitted(name), (f"reference emitted {name}_b (codegen.cpp:332-382), gcc "
                                   f"{ref_emitted_opt(name)} -fopenmp, fp64")
    f = family(name)

    def view(a):
        return a.numpy() if hasattr(a, "numpy") else a

    def call(n, scalars, arrays):
        grids = {a: view(arrays[a]) for a in f.arrays if a in arrays}
        adjs = {b: view(arrays[b]) for b in f.adjoints if b and b in arrays}
        rc = run_program_omp(name, n, scalars, grids, adjs)
        return 0 if rc >= 1 else 1
    return call, (f"oracle port sg_run_program_omp (restates interp.cpp:189-198; pinned to "
                  f"the reference by tests/test_oracle_pins.py), fp64 -- "
                  f"oracle/_ref/libref_{name}.so not built here")


def ref_emitted(name: str, kind: str = "adjoint"):
    """The reference's OWN generated OpenMP function (emit_primal /
    emit_adjoint / emit_scatter_adjoint, codegen.cpp:311-434, compiled by
    oracle/ref/Makefile into oracle/_ref/libref_<name>.so).  Returns
    call(n, scalars, arrays) -> return code, arrays = name -> C-contiguous
    fp64 buffer (numpy array or CPU torch tensor), updated in place."""
    fn_name = name + {"primal": "", "adjoint": "_b", "scatter": "_scatter_b"}[kind]
    if name not in _ref_libs:
        _ref_libs[name] = ctypes.CDLL(ref_emitted_path(name))
    fn = getattr(_ref_libs[name], fn_name)
    fn.restype = ctypes.c_int
    params = _ref_params(name, fn_name)

    def ptr(a):
        if hasattr(a, "data_ptr"):
            import torch
            assert a.dtype == torch.float64 and a.is_contiguous() and not a.is_cuda
            return ctypes.c_void_p(a.data_ptr())
        assert a.dtype == np.float64 and a.flags.c_contiguous
        return ctypes.c_void_p(a.ctypes.data)

    def call(n, scalars, arrays):
        args = []
        for typ, pn in params:
            if typ == "int":
                args.append(ctypes.c_int(int(n) if pn == "n" else int(scalars[pn])))
            elif typ == "double":
                args.append(ctypes.c_double(float(scalars[pn])))
            else:
                args.append(ptr(arrays[pn]))
        return fn(*args)
    call.params = [pn for typ, pn in params if typ == "ptr"]
    return call
