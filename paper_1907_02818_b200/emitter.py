"""CUDA back-end emitter for arbitrary adjoint-stencil programs.

The reference turns an ``AdjointProgram`` into C/OpenMP text with
``emit_adjoint`` (codegen.cpp:332-382).  This module turns the same program
-- the primal spec (counters, affine bounds, arrays, lhs, rhs) plus the
derived terms (active read, offset, partial S_l printed by the reference's
``to_input_string``, expr.cpp:261-397) -- into CUDA C for sm_100a, compiled at
run time with NVRTC through the C ABI (``sgb_jit_compile`` / ``sgb_jit_launch``).

Emitted gather kernel (one thread per point y of the write box):

    for each target adjoint array A:
        for l in ascending term order with target A:       (adjoint.cpp:85)
            if y - o_l in B:  cell += S_l(y - o_l) * seed[perm(y - o_l)]
        store cell if any term reached y                   (untouched otherwise)

i.e. the predicate form of the reference's hierarchical core + boundary nests
(SURVEY Appendix C), with the per-cell increments in the same order as
``run_program`` (interp.cpp:153-198).  The primal kernel mirrors ``run_nest``.
This general path covers every problem the front end accepts (lap1d,
burgers1d, wave3d, the config families, the reference's fuzz problems); the
hand-tuned TMA kernels remain the hot path for the BASELINE configs.
"""
from __future__ import annotations

import ctypes
import json
import re

import numpy as np
from dataclasses import dataclass

from . import _lib

# ------------------------------------------------------------------ parsing
_TOK = re.compile(r"\s*(?:(\d+\.\d*(?:[eE][-+]?\d+)?|\d+(?:[eE][-+]?\d+)?|\.\d+(?:[eE][-+]?\d+)?)"
                  r"|([A-Za-z_]\w*)|(>=|<=|[-+*/(),\[\]<>=]))")


def _tokens(text):
    pos, out = 0, []
    text = text.strip()
    while pos < len(text):
        m = _TOK.match(text, pos)
        if not m or m.end() == pos:
            raise ValueError(f"cannot tokenize {text[pos:]!r}")
        num, ident, op = m.groups()
        out.append(("num", num) if num else ("id", ident) if ident else ("op", op))
        pos = m.end()
    return out


class _Parser:
    """Precedence climbing over the reference's expression syntax
    (parser.cpp:11-225 accepts it; to_input_string prints it)."""

    def __init__(self, text):
        self.t = _tokens(text)
        self.i = 0

    def peek(self):
        return self.t[self.i] if self.i < len(self.t) else (None, None)

    def at(self, k):
        """Value of the token k positions ahead (None past the end)."""
        j = self.i + k
        return self.t[j][1] if j < len(self.t) else None

    def take(self, val=None):
        tok = self.peek()
        if val is not None and tok[1] != val:
            raise ValueError(f"expected {val!r}, got {tok}")
        self.i += 1
        return tok

    def parse(self):
        e = self.compare()
        if self.i != len(self.t):
            raise ValueError(f"trailing input at token {self.t[self.i]}")
        return e

    def compare(self):
        a = self.additive()
        if self.peek()[1] in (">=", "<=", ">", "<"):
            op = self.take()[1]
            return ("cmp", op, a, self.additive())
        return a

    def additive(self):
        e = self.term()
        while self.peek()[1] in ("+", "-"):
            op = self.take()[1]
            e = ("add" if op == "+" else "sub", e, self.term())
        return e

    def term(self):
        e = self.unary()
        while self.peek()[1] in ("*", "/"):
            op = self.take()[1]
            e = ("mul" if op == "*" else "div", e, self.unary())
        return e

    def unary(self):
        if self.peek()[1] == "-":
            self.take()
            return ("neg", self.unary())
        if self.peek()[1] == "+":
            self.take()
            return self.unary()
        return self.atom()

    def atom(self):
        kind, val = self.take()
        if kind == "num":
            return ("num", val)
        if kind == "op" and val == "(":
            e = self.compare()
            self.take(")")
            return e
        if kind == "id":
            if val == "derivative" and self.peek()[1] == "(":
                # OpaqueDeriv as printed by to_input_string (expr.cpp:374-388):
                # derivative(f, a)(a=<expr>, b=<expr>) -> call f_d_a(...)
                self.take("(")
                fn = self.take()[1]
                self.take(",")
                wrt = self.take()[1]
                self.take(")")
                return ("opaque", f"{fn}_d_{wrt}", self.kwargs())
            if self.peek()[1] == "(" and self.at(2) == "=":
                return ("opaque", val, self.kwargs())  # OpaqueCall f(a=.., b=..)
            if self.peek()[1] == "(":
                self.take("(")
                args = [self.compare()]
                while self.peek()[1] == ",":
                    self.take(",")
                    args.append(self.compare())
                self.take(")")
                if val in ("max", "min") and len(args) == 2:
                    return (val, args[0], args[1])
                if val == "pow" and len(args) == 2:
                    k = args[1]
                    sign = 1
                    if k[0] == "neg":
                        sign, k = -1, k[1]
                    if k[0] != "num" or not re.fullmatch(r"\d+", k[1]):
                        raise ValueError("pow exponent must be an integer literal")
                    return ("pow", args[0], sign * int(k[1]))
                if val == "select" and len(args) == 3 and args[0][0] == "cmp":
                    return ("select", args[0], args[1], args[2])
                raise ValueError(f"unsupported call {val}/{len(args)} (opaque calls take "
                                 "named arguments: {val}(a=..., b=...))")
            if self.peek()[1] == "[":
                idx = []
                while self.peek()[1] == "[":
                    self.take("[")
                    c = self.take()
                    if c[0] != "id":
                        raise ValueError("array index must start with a counter")
                    off = 0
                    if self.peek()[1] in ("+", "-"):
                        sgn = 1 if self.take()[1] == "+" else -1
                        off = sgn * int(self.take()[1])
                    self.take("]")
                    idx.append((c[1], off))
                return ("read", val, idx)
            return ("sym", val)
        raise ValueError(f"unexpected token {val!r}")


    def kwargs(self):
        """(name=expr, ...) argument list of an opaque call, in printed
        (argument-name) order, which is also the C call order
        (codegen.cpp:153-168)."""
        self.take("(")
        out = []
        while True:
            name = self.take()[1]
            self.take("=")
            out.append((name, self.compare()))
            if self.peek()[1] != ",":
                break
            self.take(",")
        self.take(")")
        return out


def parse_expr(text):
    return _Parser(text).parse()


def parse_affine(text):
    """'n - 2' -> ({'n': 1}, -2) (AffineExpr, affine.cpp:81-200)."""
    coeff, const = {}, 0
    e = parse_expr(text)

    def walk(node, sign):
        nonlocal const
        k = node[0]
        if k == "num":
            const += sign * int(node[1])
        elif k == "sym":
            coeff[node[1]] = coeff.get(node[1], 0) + sign
        elif k == "add":
            walk(node[1], sign)
            walk(node[2], sign)
        elif k == "sub":
            walk(node[1], sign)
            walk(node[2], -sign)
        elif k == "neg":
            walk(node[1], -sign)
        elif k == "mul" and node[1][0] == "num":
            inner_c, inner_k = parse_affine_node(node[2])
            f = int(node[1][1]) * sign
            for s_, v in inner_c.items():
                coeff[s_] = coeff.get(s_, 0) + f * v
            const += f * inner_k
        else:
            raise ValueError(f"non-affine bound {text!r}")
    walk(e, 1)
    return coeff, const


def parse_affine_node(node):
    c, k = {}, 0
    if node[0] == "sym":
        c[node[1]] = 1
    elif node[0] == "num":
        k = int(node[1])
    else:
        raise ValueError("non-affine")
    return c, k


def affine_c(aff, sizes_var):
    coeff, const = aff
    parts = [f"({v} * {sizes_var[s]})" for s, v in coeff.items()]
    # plain int literal: the arithmetic takes the size variables' type
    # (I = int or long long), so a 32-bit kernel stays 32-bit
    lit = f"({const})" if -2 ** 31 < const < 2 ** 31 else f"({const}LL)"
    return "(" + " + ".join(parts + [lit]) + ")"


# ------------------------------------------------------------------ codegen
@dataclass
class Term:
    array: str
    adjoint: str
    offset: tuple
    partial: str


class _CGen:
    def __init__(self, prob, counters, at, flat=None):
        self.p = prob
        self.counters = counters  # counter name -> C expression of its value
        self.at = at              # array name -> C flat-index function name
        # flat addressing (gather): {"shift": {counter: s}, "arrays": set} -- a
        # read A[c_0 + k_0]..[c_r + k_r] of an array laid out in counter order
        # at x = y + shift is fy_A + sum_i (k_i + shift_i) * sd_A_i
        self.flat = flat

    def e(self, node):
        k = node[0]
        if k == "num":
            v = node[1]
            return f"T({v})" if ("." in v or "e" in v or "E" in v) else f"T({v}.0)"
        if k == "sym":
            if node[1] not in self.p.scalars:
                raise ValueError(f"unknown scalar {node[1]}")
            return f"s_{node[1]}"
        if k == "read":
            name, idx = node[1], node[2]
            if self.flat is not None and name in self.flat["arrays"] and \
                    [c for c, _ in idx] == self.p.counters:
                sh = self.flat["shift"]
                r = len(idx)
                terms = []
                for dim, (c, o) in enumerate(idx):
                    dd = o + sh[c]
                    if dd:
                        terms.append(f"{dd}" if dim == r - 1 else f"({dd}) * sd_{name}_{dim}")
                off = " + ".join(terms)
                return f"a_{name}[fy_{name}" + (f" + ({off})" if off else "") + "]"
            args = ", ".join(f"({self.counters[c]} + ({o}))" for c, o in idx)
            return f"a_{name}[{self.at[name]}({args})]"
        if k in ("add", "sub", "mul", "div"):
            op = {"add": "+", "sub": "-", "mul": "*", "div": "/"}[k]
            return f"({self.e(node[1])} {op} {self.e(node[2])})"
        if k == "neg":
            return f"(-{self.e(node[1])})"
        if k == "max":
            return f"fmax({self.e(node[1])}, {self.e(node[2])})"
        if k == "min":
            return f"fmin({self.e(node[1])}, {self.e(node[2])})"
        if k == "pow":
            base, p_ = self.e(node[1]), node[2]
            return f"ipow({base}, {p_})"
        if k == "select":
            c = node[1]
            return f"(({self.e(c[2])} {c[1]} {self.e(c[3])}) ? {self.e(node[2])} : {self.e(node[3])})"
        if k == "cmp":
            raise ValueError("comparison outside select")
        if k == "opaque":
            # user-supplied __device__ function (EmittedProblem(device_functions=)),
            # arguments positional in argument-name order like the reference's C
            return f"{node[1]}(" + ", ".join(self.e(x) for _, x in node[2]) + ")"
        raise ValueError(k)


class EmittedProblem:
    """A reference problem (spec dict + terms) lowered to sm_100a kernels."""

    def __init__(self, spec: dict, terms, dtype: str = "f64", device_functions: str = ""):
        """`device_functions`: CUDA source defining every opaque function and
        derivative the program calls (e.g. ``__device__ T f_d_a(T a, T b)``,
        T = the kernel's element type) -- the device counterpart of the
        reference's `EmitOptions.opaque_prototypes` (codegen.hpp:17-18)."""
        self.spec = spec
        self.device_functions = device_functions
        self.name = spec["name"]
        self.counters = list(spec["counters"])
        self.d = len(self.counters)
        self.sizes = list(spec["sizes"])
        self.scalars = list(spec["scalars"])
        self.bounds = [(parse_affine(spec["bounds"][c][0]), parse_affine(spec["bounds"][c][1]))
                       for c in self.counters]
        self.arrays = {}  # declaration order
        for name, a in spec["arrays"].items():
            self.arrays[name] = {"shape": [parse_affine(x) for x in a["shape"]],
                                 "active": bool(a.get("active")), "adjoint": a.get("adjoint"),
                                 "role": a.get("role", "input")}
        m = re.fullmatch(r"\s*(\w+)((?:\[\s*\w+\s*\])+)\s*", spec["lhs"])
        self.out = m.group(1)
        self.lhs = re.findall(r"\[\s*(\w+)\s*\]", m.group(2))
        self.seed = self.arrays[self.out]["adjoint"]
        self.increment = spec.get("mode", "=") == "+="
        self.rhs = parse_expr(spec["rhs"])
        self.terms = [t if isinstance(t, Term) else
                      Term(t["array"], t["adjoint"], tuple(t["offset"]), t["partial"])
                      for t in terms]
        self.partials = [parse_expr(t.partial) for t in self.terms]
        self.T = {"f64": "double", "f32": "float"}[dtype]
        self.dtype = dtype
        self._kern = {}
        self._which = "all"

    # -- names and ABI order (codegen.cpp:198-211: declaration order, each
    #    primal followed by its adjoint)
    def param_arrays(self, which="all"):
        """Arrays of a kernel's signature in the reference's ABI order: every
        REFERENCED array in declaration order, each primal followed by its
        adjoint (collect_refs, codegen.cpp:198-211)."""
        def reads(node, acc):
            if isinstance(node, tuple):
                if node and node[0] == "read":
                    acc.add(node[1])
                for x in node[1:]:
                    reads(x, acc)
            elif isinstance(node, list):  # opaque-call arguments
                for x in node:
                    reads(x, acc)
            return acc
        used = set()
        if which in ("gather", "nest", "all"):
            for part in self.partials:
                reads(part, used)
            used.update(t.adjoint for t in self.terms)
            used.add(self.seed)
        if which in ("primal", "all"):
            reads(self.rhs, used)
            used.add(self.out)
        out = []
        for name, a in self.arrays.items():
            if name in used:
                out.append(name)
            if a["active"] and a["adjoint"] in used:
                out.append(a["adjoint"])
        return out

    def _shape_of(self, arr):
        for name, a in self.arrays.items():
            if arr == name or arr == a["adjoint"]:
                return a["shape"]
        raise KeyError(arr)

    def _prelude(self, index="long long"):
        szv = {s: f"z_{s}" for s in self.sizes}
        lines = [f"typedef {self.T} T;", f"typedef {index} I;",
                 "__device__ __forceinline__ T ipow(T b, int p) {",
                 "  T r = T(1); int q = p < 0 ? -p : p;",
                 "  for (int i = 0; i < q; i++) r *= b;",
                 "  return p < 0 ? T(1) / r : r; }"]
        if self.device_functions:
            lines.append(self.device_functions)
        # flat index per array (row-major over its own shape)
        fns = {}
        for arr in self.param_arrays(self._which):
            shp = self._shape_of(arr)
            r = len(shp)
            args = ", ".join(f"I x{i}" for i in range(r))
            body = "x0"
            for i in range(1, r):
                body = f"(({body}) * {affine_c(shp[i], szv)} + x{i})"
            fn = f"ix_{arr}"
            fns[arr] = fn
            lines.append(f"__device__ __forceinline__ I {fn}({args}, "
                         + ", ".join(f"I z_{s}" for s in self.sizes) + f") {{ return {body}; }}")
        return lines, fns, szv

    def _written(self):
        """Arrays the current kernel writes (the gather / nest forms: the
        adjoint targets; the primal: its output); the rest are passed as
        const __restrict__, so their loads may take the read-only path."""
        if self._which == "primal":
            return {self.out}
        return {t.adjoint for t in self.terms}

    def _signature(self, kname, index="long long"):
        ps = [f"{index} z_{s}" for s in self.sizes]
        ps += [f"T s_{s}" for s in self.scalars]
        written = self._written()
        for arr in self.param_arrays(self._which):
            q = "" if arr in written else "const "
            ps.append(f"{q}T* __restrict__ a_{arr}")
        return f'extern "C" __global__ void {kname}(' + ", ".join(ps) + ")"

    def _box_checks(self, xs, szv):
        conds = []
        for i, (lo, hi) in enumerate(self.bounds):
            conds.append(f"({xs[i]} >= {affine_c(lo, szv)} && {xs[i]} <= {affine_c(hi, szv)})")
        return " && ".join(conds) if conds else "true"

    def _write_box(self, szv):
        """Union of the target adjoint arrays' extents (per dimension)."""
        ext = []
        for i in range(self.d):
            cands = []
            for t in self.terms:
                c = affine_c(self._shape_of(t.adjoint)[i], szv)
                if c not in cands:
                    cands.append(c)
            e = cands[0]
            for c in cands[1:]:
                e = f"max({e}, {c})"
            ext.append(e)
        return ext

    def _unroll(self):
        import os
        return max(1, int(os.environ.get("SGB_EMIT_UNROLL", "2"))) if self.d >= 3 else 1

    def gather_source(self, index="long long"):
        """Fused predicated gather.  Threads map to (.., j, k) = (z, y, x) of a
        3D launch with grid-stride outer loops (no div/mod); per target array
        a point inside the target's core box -- the intersection of its terms'
        valid boxes B + o_l -- applies every term unpredicated, any other point
        tests each term (same per-cell order either way, so bitwise equal)."""
        self._which = "gather"
        lines, fns, szv = self._prelude(index)
        zargs = ", ".join(f"z_{s}" for s in self.sizes)
        at = {arr: f"AT_{arr}" for arr in self.param_arrays(self._which)}
        for arr, fn in fns.items():
            lines.append(f"#define AT_{arr}(...) {fn}(__VA_ARGS__, {zargs})")
        lines.append(self._signature("sgb_emitted_gather", index) + " {")
        ext = self._write_box(szv)
        for i in range(self.d):
            lines.append(f"  const I W{i} = {ext[i]};")
        d = self.d
        # arrays laid out in counter order (rank d): flat base index per point
        # plus per-dimension strides, so every shifted read is base + const
        flat_arrays = [a for a in self.param_arrays(self._which)
                       if len(self._shape_of(a)) == d]
        for a in flat_arrays:
            shp = self._shape_of(a)
            for dim in range(d - 1):
                st = " * ".join(affine_c(shp[q], szv) for q in range(dim + 1, d))
                lines.append(f"  const I sd_{a}_{dim} = {st};")
        inner = d - 1
        lines.append(f"  const I y{inner} = blockIdx.x * (I)blockDim.x + threadIdx.x;")
        lines.append(f"  if (y{inner} >= W{inner}) return;")
        depth = 1
        if d >= 2:
            lines.append(f"  for (I y{d - 2} = blockIdx.y * (I)blockDim.y + threadIdx.y; "
                         f"y{d - 2} < W{d - 2}; y{d - 2} += gridDim.y * (I)blockDim.y) {{")
            depth += 1
        if d >= 3:
            # UF consecutive outer-dimension points per thread, unrolled, so
            # their independent load streams overlap (memory-level parallelism)
            uf = self._unroll()
            lines.append(f"  for (I yb = (blockIdx.z * (I)blockDim.z + threadIdx.z) * {uf}; "
                         f"yb < W{d - 3}; yb += gridDim.z * (I)blockDim.z * {uf}) {{")
            lines.append("#pragma unroll")
            lines.append(f"  for (int uu = 0; uu < {uf}; uu++) {{")
            lines.append(f"  const I y{d - 3} = yb + uu;")
            lines.append(f"  if (y{d - 3} < W{d - 3}) {{")
            depth += 3
        # group terms by target adjoint, ascending term order inside each
        targets = []
        for t in self.terms:
            if t.adjoint not in targets:
                targets.append(t.adjoint)
        cidx = {c: i for i, c in enumerate(self.counters)}
        ys = ", ".join(f"y{i}" for i in range(d))
        for a in flat_arrays:
            lines.append(f"  const I fy_{a} = AT_{a}({ys});")
        for tgt in targets:
            shp = self._shape_of(tgt)
            inb = " && ".join(f"y{i} < {affine_c(shp[i], szv)}" for i in range(d))
            mine = [(ti, t, part) for ti, (t, part) in enumerate(zip(self.terms, self.partials))
                    if t.adjoint == tgt]
            core = []
            for i in range(d):
                lo, hi = self.bounds[i]
                omax = max(t.offset[i] for _, t, _ in mine)
                omin = min(t.offset[i] for _, t, _ in mine)
                core.append(f"y{i} >= {affine_c(lo, szv)} + ({omax}) && "
                            f"y{i} <= {affine_c(hi, szv)} + ({omin})")
            lines.append(f"  if ({inb}) {{")
            lines.append(f"    if ({' && '.join(core)}) {{  // core of {tgt}: every term valid")
            tix = f"fy_{tgt}" if tgt in flat_arrays else f"AT_{tgt}({ys})"
            lines.append(f"      T cell = a_{tgt}[{tix}];")
            exprs = []
            for ti, t, part in mine:
                xs = [f"(y{i} - ({t.offset[i]}))" for i in range(d)]
                flat = {"shift": {c: -t.offset[cidx[c]] for c in self.counters},
                        "arrays": set(flat_arrays)}
                cg = _CGen(self, {c: xs[cidx[c]] for c in self.counters}, at, flat)
                seed_read = ("read", self.seed, [(c, 0) for c in self.lhs])
                exprs.append((ti, t, xs, f"({cg.e(part)}) * {cg.e(seed_read)}"))
            for ti, t, xs, ex in exprs:
                lines.append(f"      cell += {ex};  // term {ti}")
            lines.append(f"      a_{tgt}[{tix}] = cell;")
            lines.append("    } else {")
            lines.append("      bool touched = false; T cell = T(0);")
            for ti, t, xs, ex in exprs:
                lines.append(f"      if ({self._box_checks(xs, szv)}) {{  // term {ti}: "
                             f"{t.array}{list(t.offset)}")
                lines.append(f"        if (!touched) {{ cell = a_{tgt}[{tix}]; touched = true; }}")
                lines.append(f"        cell += {ex};")
                lines.append("      }")
            lines.append(f"      if (touched) a_{tgt}[{tix}] = cell;")
            lines.append("    }")
            lines.append("  }")
        lines.append("  }" * (depth - 1))
        lines.append("}")
        return "\n".join(lines) + "\n"

    def nest_source(self):
        self._which = "nest"
        """The reference's structure (adjoint.cpp:73-150): one kernel applied to
        ONE hierarchical nest per launch -- box [lo, hi] and the nest's term
        set as a bitmask, no per-point predicate (the nest guarantees every
        listed term is valid).  Boundary-strategy A/B against the fused form."""
        lines, fns, szv = self._prelude()
        zargs = ", ".join(f"z_{s}" for s in self.sizes)
        at = {arr: f"AT_{arr}" for arr in self.param_arrays(self._which)}
        for arr, fn in fns.items():
            lines.append(f"#define AT_{arr}(...) {fn}(__VA_ARGS__, {zargs})")
        sig = self._signature("sgb_emitted_nest")[:-1]
        sig += ", " + ", ".join(f"long long lo{i}, long long hi{i}" for i in range(self.d))
        sig += ", unsigned long long mask)"
        lines.append(sig + " {")
        lines.append("  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;")
        for i in range(self.d):
            lines.append(f"  const long long N{i} = hi{i} - lo{i} + 1;")
        total = " * ".join(f"N{i}" for i in range(self.d))
        lines.append(f"  if (t >= {total}) return;")
        for i in reversed(range(self.d)):
            if i == 0:
                lines.append("  const long long y0 = lo0 + t;")
            else:
                lines.append(f"  const long long y{i} = lo{i} + t % N{i}; t /= N{i};")
        cidx = {c: i for i, c in enumerate(self.counters)}
        ys = ", ".join(f"y{i}" for i in range(self.d))
        for ti, (t, part) in enumerate(zip(self.terms, self.partials)):
            xs = [f"(y{i} - ({t.offset[i]}))" for i in range(self.d)]
            cg = _CGen(self, {c: xs[cidx[c]] for c in self.counters}, at)
            seed_idx = ", ".join(xs[cidx[c]] for c in self.lhs)
            lines.append(f"  if (mask & (1ULL << {ti}))  // term {ti}")
            lines.append(f"    a_{t.adjoint}[AT_{t.adjoint}({ys})] += ({cg.e(part)}) * "
                         f"a_{self.seed}[AT_{self.seed}({seed_idx})];")
        lines.append("}")
        return "\n".join(lines) + "\n"

    def nests(self, sizes):
        """Hierarchical core + boundary nests (Splitter::recurse,
        adjoint.cpp:73-120) at concrete sizes: [(lo[], hi[], term indices)]."""
        offs = [t.offset for t in self.terms]
        lo = [self._eval_aff(b[0], sizes) for b in self.bounds]
        hi = [self._eval_aff(b[1], sizes) for b in self.bounds]
        out = []

        def rec(dim, plo, phi, alive):
            if dim == self.d:
                out.append((list(plo), list(phi), list(alive)))
                return
            ds = sorted({offs[a][dim] for a in alive})
            k = len(ds)
            s_, e_ = lo[dim], hi[dim]
            for j in range(k - 1):
                rec(dim + 1, plo + [s_ + ds[j]], phi + [s_ + ds[j + 1] - 1],
                    [a for a in alive if offs[a][dim] <= ds[j]])
            rec(dim + 1, plo + [s_ + ds[-1]], phi + [e_ + ds[0]], alive)
            for j in range(k - 1):
                rec(dim + 1, plo + [e_ + ds[j] + 1], phi + [e_ + ds[j + 1]],
                    [a for a in alive if offs[a][dim] > ds[j]])
        rec(0, [], [], list(range(len(self.terms))))
        return out

    def primal_source(self):
        self._which = "primal"
        lines, fns, szv = self._prelude()
        zargs = ", ".join(f"z_{s}" for s in self.sizes)
        at = {arr: f"AT_{arr}" for arr in self.param_arrays(self._which)}
        for arr, fn in fns.items():
            lines.append(f"#define AT_{arr}(...) {fn}(__VA_ARGS__, {zargs})")
        lines.append(self._signature("sgb_emitted_primal") + " {")
        lines.append("  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;")
        for i, (lo, hi) in enumerate(self.bounds):
            lines.append(f"  const long long L{i} = {affine_c(lo, szv)}, "
                         f"N{i} = {affine_c(hi, szv)} - L{i} + 1;")
            lines.append(f"  if (N{i} <= 0) return;")
        total = " * ".join(f"N{i}" for i in range(self.d))
        lines.append(f"  if (t >= {total}) return;")
        for i in reversed(range(self.d)):
            if i == 0:
                lines.append("  const long long x0 = L0 + t;")
            else:
                lines.append(f"  const long long x{i} = L{i} + t % N{i}; t /= N{i};")
        xs = {c: f"x{i}" for i, c in enumerate(self.counters)}
        cg = _CGen(self, xs, at)
        lidx = ", ".join(xs[c] for c in self.lhs)
        op = "+=" if self.increment else "="
        lines.append(f"  a_{self.out}[AT_{self.out}({lidx})] {op} {cg.e(self.rhs)};")
        lines.append("}")
        return "\n".join(lines) + "\n"

    # ------------------------------------------------------------ run
    def check_compiles(self):
        """NVRTC-compile both kernels for sm_100a without loading them (no GPU
        needed); raises StencilError with the compiler log on failure."""
        for src in (self.gather_source(), self.primal_source()):
            if _lib.lib().sgb_jit_check(src.encode()) != 0:
                raise _lib.StencilError(_lib.lib().sgb_jit_log().decode())

    def _kernel(self, which, index="long long"):
        key = (which, index)
        if key not in self._kern:
            if which == "gather":
                src = self.gather_source(index)
            else:
                src = {"primal": self.primal_source, "nest": self.nest_source}[which]()
            h = ctypes.c_void_p()
            rc = _lib.lib().sgb_jit_compile(src.encode(), f"sgb_emitted_{which}".encode(),
                                            ctypes.byref(h))
            if rc != 0:
                raise _lib.StencilError(_lib.lib().sgb_last_error().decode())
            self._kern[key] = h
        return self._kern[key]

    def _launch(self, which, sizes, scalars, arrays, nthreads, stream=None, extra=(),
                grid=None, index="long long"):
        import torch
        from .api import _stream_ptr
        keep = []
        argv = []
        for s in self.sizes:
            v = (ctypes.c_int if index == "int" else ctypes.c_longlong)(int(sizes[s]))
            keep.append(v)
        T = ctypes.c_double if self.T == "double" else ctypes.c_float
        for s in self.scalars:
            keep.append(T(float(scalars.get(s, 0.0))))
        tdt = torch.float64 if self.T == "double" else torch.float32
        for arr in self.param_arrays("primal" if which == "primal" else "gather"):
            t = arrays.get(arr)
            if t is None:
                raise _lib.StencilError(f"{self.name}: missing array {arr}")
            if not (t.is_cuda and t.is_contiguous() and t.dtype == tdt):
                raise _lib.StencilError(f"{arr}: contiguous CUDA {tdt} tensor required")
            keep.append(ctypes.c_void_p(t.data_ptr()))
        keep.extend(extra)
        argv = (ctypes.c_void_p * len(keep))(*[ctypes.cast(ctypes.pointer(k), ctypes.c_void_p)
                                               for k in keep])
        if grid is None:
            blocks = max(1, (nthreads + 255) // 256)
            if blocks > 2 ** 31 - 1:
                raise _lib.StencilError("grid too large")
            grid = (blocks, 1, 1, 256, 1, 1)
        rc = _lib.lib().sgb_jit_launch(self._kernel(which, index), *grid, argv,
                                       _stream_ptr(stream))
        _lib.check(rc, f"{self.name} emitted {which}")

    def _eval_aff(self, aff, sizes):
        coeff, const = aff
        return const + sum(v * int(sizes[s]) for s, v in coeff.items())

    def guards_ok(self, sizes) -> bool:
        """Minimum-extent guards of split_regions (adjoint.cpp:134-143)."""
        for i in range(self.d):
            offs = [t.offset[i] for t in self.terms]
            if not offs:
                continue
            span = max(offs) - min(offs)
            lo, hi = self.bounds[i]
            if span >= 1 and self._eval_aff(hi, sizes) - self._eval_aff(lo, sizes) < span:
                return False
        return True

    def adjoint(self, sizes, scalars, arrays, stream=None):
        """Gather adjoint (+= into every adjoint array) on the device."""
        if not self.terms:
            return
        if not self.guards_ok(sizes):
            raise _lib.GuardViolation(f"{self.name}: minimum extent violated")
        W = [max(self._eval_aff(self._shape_of(t.adjoint)[i], sizes) for t in self.terms)
             for i in range(self.d)]
        # 32-bit indices when every referenced array fits
        big = max(int(np.prod([self._eval_aff(a, sizes) for a in self._shape_of(arr)]))
                  for arr in self.param_arrays("gather"))
        index = "int" if big < 2 ** 31 - 1 else "long long"
        bx = 32 if self.d > 1 else 256
        by = 8 if self.d > 1 else 1
        gx = (W[-1] + bx - 1) // bx
        gy = min((W[-2] + by - 1) // by, 65535) if self.d >= 2 else 1
        gz = min((W[0] + self._unroll() - 1) // self._unroll(), 65535) if self.d >= 3 else 1
        if gx > 2 ** 31 - 1:
            raise _lib.StencilError("grid too large")
        self._launch("gather", sizes, scalars, arrays, 0, stream,
                     grid=(max(1, gx), max(1, gy), max(1, gz), bx, by, 1), index=index)

    def adjoint_nests(self, sizes, scalars, arrays, nests=None, stream=None):
        """The same adjoint as `adjoint`, executed the reference's way: one
        launch per hierarchical nest, in program order.  Returns #launches."""
        if not self.guards_ok(sizes):
            raise _lib.GuardViolation(f"{self.name}: minimum extent violated")
        if len(self.terms) > 64:
            raise _lib.StencilError("nest form supports up to 64 terms")
        count = 0
        for lo, hi, terms in (nests if nests is not None else self.nests(sizes)):
            pts = 1
            for a, b in zip(lo, hi):
                pts *= max(0, b - a + 1)
            if pts == 0 or not terms:
                continue
            mask = 0
            for t in terms:
                mask |= 1 << t
            extra = []
            for a, b in zip(lo, hi):
                extra += [ctypes.c_longlong(a), ctypes.c_longlong(b)]
            extra.append(ctypes.c_ulonglong(mask))
            self._launch("nest", sizes, scalars, arrays, pts, stream, extra)
            count += 1
        return count

    def primal(self, sizes, scalars, arrays, stream=None):
        total = 1
        for lo, hi in self.bounds:
            total *= max(0, self._eval_aff(hi, sizes) - self._eval_aff(lo, sizes) + 1)
        if total:
            self._launch("primal", sizes, scalars, arrays, total, stream)


def from_reference_info(spec: dict, info: dict, dtype="f64") -> EmittedProblem:
    """Build from the reference's own program structure (`ref_harness info`:
    terms in active_reads order with to_input_string partials)."""
    return EmittedProblem(spec, info["terms"], dtype)


def load_program(family: str, dtype: str = "f64") -> EmittedProblem:
    """A committed front-end output (programs/<family>.json) as an emitted problem."""
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "programs",
                           family + ".json")) as fh:
        d = json.load(fh)
    return EmittedProblem(d["spec"], d["terms"], dtype)


def load_spec(path: str) -> dict:
    with open(path) as fh:
        return json.load(fh)
