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
        if k in ("add", "sub") and getattr(self.p, "fma", False):
            # a + b*c -> fma(b, c, a), a - b*c -> fma(-b, c, a), b*c + a ->
            # fma(b, c, a): written out, so every emitted form (per nest,
            # fused, tiled, primal) rounds each sum of products identically
            # (the kernels are compiled --fmad=false: no implicit contraction)
            L, Rn = node[1], node[2]
            if Rn[0] == "mul":
                b = self.e(Rn[1])
                return (f"fma({b}, {self.e(Rn[2])}, {self.e(L)})" if k == "add" else
                        f"fma(-({b}), {self.e(Rn[2])}, {self.e(L)})")
            if k == "add" and L[0] == "mul":
                return f"fma({self.e(L[1])}, {self.e(L[2])}, {self.e(Rn)})"
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


def _reads(node, out):
    """Every ("read", name, idx) in an expression tree, in tree order."""
    if isinstance(node, tuple):
        if node and node[0] == "read":
            out.append(node)
        for x in node[1:]:
            _reads(x, out)
    elif isinstance(node, list):  # opaque-call arguments (name, node)
        for x in node:
            _reads(x, out)
    return out


class _RingCGen(_CGen):
    """_CGen whose counter-aligned reads of ring fields come from the tiled
    kernel's shared-memory planes: a read at point y + r (r relative to the
    output point y of the thread) is sh_<f>[slot(y0 + r0)][ly + r1 - lo1][lx +
    r2 - lo2]; every other read is a global (flat) load as in the base class."""

    def __init__(self, prob, counters, at, flat, ring, shift):
        super().__init__(prob, counters, at, flat)
        self.ring = ring    # array name -> field dict
        self.shift = shift  # counter -> shift of this evaluation point vs y

    def e(self, node):
        if node[0] == "read" and node[1] in self.ring and \
                [c for c, _ in node[2]] == self.p.counters:
            f = self.ring[node[1]]
            r = [o + self.shift[c] for c, o in node[2]]
            return _ring_ref(f, r)
        return super().e(node)


class _RegCGen(_CGen):
    """_CGen whose reads are registers already holding the value (the tiled
    gather's prefetched plane)."""

    def __init__(self, prob, counters, at, regs):
        super().__init__(prob, counters, at)
        self.regs = regs  # repr(read node) -> register name

    def e(self, node):
        if node[0] == "read":
            return self.regs[repr(node)]
        return super().e(node)


def _ring_ref(f, r):
    """Shared-memory element of field f at relative position r (the slot of
    plane y0 + r0 is s_<r0> in the kernel)."""
    row = f"(lr + ({r[1] - f['lo'][1]}))"
    col = f"(lx + ({r[2] - f['lo'][2]}))"
    return (f"sh_{f['name']}[(s_{_zn(r[0])} * {f['by']} + {row}) * {f['bx']} + {col}]")


def _zn(k):
    return f"m{-k}" if k < 0 else f"p{k}"


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
        self._factorise()
        self.T = {"f64": "double", "f32": "float"}[dtype]
        # explicit fused multiply-adds for a + b*c in every emitted form
        # (SGB_EMIT_FMA=0: separate multiply and add, the reference C's rounding)
        import os
        self.fma = os.environ.get("SGB_EMIT_FMA", "1") != "0"
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

    # -- common-subexpression factoring of the partials
    @staticmethod
    def _is_const(node):
        return node[0] == "num" or (node[0] == "neg" and node[1][0] == "num")

    def _factorise(self):
        """S_l = k_l * F_l with k_l a numeric literal (the leading factor of
        the partial's left-associated product; k_l = 1 when there is none,
        F_l = S_l) -- the wave stencils' partials
        w.r.t. the shifted u reads are all `w_l * D * c^2`.  Terms whose F_l
        coincide form a group g and share Q_g(x) = F_g(x) * seed(x): every
        emitted form evaluates such a term as k_l * (F_g(x) * seed(x)) (the
        hand-tuned kernels' q = D c^2 u_b, shared by the 24 shifted terms),
        so the forms stay bitwise equal to each other; against run_program's
        (k_l * F_l) * seed the rounding differs in the last place only."""
        split = []
        for part in self.partials:
            chain, n = [], part
            while n[0] == "mul":
                chain.insert(0, n[2])
                n = n[1]
            chain.insert(0, n)
            if len(chain) >= 2 and self._is_const(chain[0]) and \
                    not any(self._is_const(c) for c in chain[1:]):
                f = chain[1]
                for c in chain[2:]:
                    f = ("mul", f, c)
                split.append((chain[0], f))
            elif self._is_const(part):
                split.append(None)     # a constant partial: nothing to share
            else:
                split.append((None, part))  # k = 1: S_l itself is shared
        by_key = {}
        for ti, sp in enumerate(split):
            if sp is not None:
                by_key.setdefault(repr(sp[1]), []).append(ti)
        self.groups = []          # [(F node, [term indices])] with >= 2 terms
        self.factor = [None] * len(self.terms)  # term -> (k node, group index)
        for key, tis in by_key.items():
            if len(tis) < 2:
                continue
            g = len(self.groups)
            self.groups.append((split[tis[0]][1], tis))
            for ti in tis:
                self.factor[ti] = (split[ti][0], g)

    def _term_update(self, cg, ti, seed_read, cell, q=None):
        """C expression of the cell value after term ti's increment (cell: the
        running value; q: the shared Q_g(y - o_l) expression in the tiled
        form).  Factored terms add k_l * Q_g with Q_g = F_g * seed rounded
        once (k_l = 1: Q_g itself), the others S_l * seed; with self.fma the
        product and the sum are one fused multiply-add, in every form alike."""
        if self.factor[ti] is not None:
            k, g = self.factor[ti]
            Q = q if q is not None else \
                f"(({cg.e(self.groups[g][0])}) * {cg.e(seed_read)})"
            if k is None:
                return f"{cell} + {Q}"
            kk = cg.e(k)
            return f"fma({kk}, {Q}, {cell})" if self.fma else f"{cell} + {kk} * {Q}"
        P, S = f"({cg.e(self.partials[ti])})", cg.e(seed_read)
        return f"fma({P}, {S}, {cell})" if self.fma else f"{cell} + {P} * {S}"

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
                exprs.append((ti, t, xs, self._term_update(cg, ti, seed_read, "cell")))
            for ti, t, xs, ex in exprs:
                lines.append(f"      cell = {ex};  // term {ti}")
            lines.append(f"      a_{tgt}[{tix}] = cell;")
            lines.append("    } else {")
            lines.append("      bool touched = false; T cell = T(0);")
            for ti, t, xs, ex in exprs:
                lines.append(f"      if ({self._box_checks(xs, szv)}) {{  // term {ti}: "
                             f"{t.array}{list(t.offset)}")
                lines.append(f"        if (!touched) {{ cell = a_{tgt}[{tix}]; touched = true; }}")
                lines.append(f"        cell = {ex};")
                lines.append("      }")
            lines.append(f"      if (touched) a_{tgt}[{tix}] = cell;")
            lines.append("    }")
            lines.append("  }")
        lines.append("  }" * (depth - 1))
        lines.append("}")
        return "\n".join(lines) + "\n"

    # -- tiled gather (3D): shared-memory planes of the factored Q fields and
    #    of the arrays the unfactored partials read at many points
    # 32 x 8 threads, TILE_Y / BLOCK_Y rows each (768^3 wave3d_r4 fp32: 8 / 16
    # / 24 / 32 rows = 9.1 / 11.9 / 13.2 / 20.6 ms, scripts/emit_tile_sweep.py)
    TILE_X, TILE_Y, BLOCK_Y = 32, 8, 8

    def tiled_layout(self):
        """Field layout of the tiled gather, or None when it does not apply
        (d != 3, targets / seed not laid out in counter order, nothing to
        share, or the planes exceed shared memory)."""
        if self.d != 3 or not self.terms or list(self.lhs) != self.counters:
            return None
        if any(len(self._shape_of(t.adjoint)) != 3 for t in self.terms):
            return None
        fields = []
        for g, (F, tis) in enumerate(self.groups):
            rs = [[-self.terms[ti].offset[i] for i in range(3)] for ti in tis]
            fields.append({"kind": "q", "g": g, "name": f"q{g}",
                           "lo": [min(r[i] for r in rs) for i in range(3)],
                           "hi": [max(r[i] for r in rs) for i in range(3)]})
        pos = {}
        for ti, t in enumerate(self.terms):
            if self.factor[ti] is not None:
                continue
            seed_read = ("read", self.seed, [(c, 0) for c in self.lhs])
            for _, name, idx in _reads(self.partials[ti], [seed_read]):
                if [c for c, _ in idx] != self.counters or len(self._shape_of(name)) != 3:
                    continue
                pos.setdefault(name, set()).add(
                    tuple(idx[i][1] - t.offset[i] for i in range(3)))
        for name, rs in sorted(pos.items()):
            if len(rs) >= 4:  # read at many points: one shared plane set
                fields.append({"kind": "raw", "name": f"r_{name}", "array": name,
                               "lo": [min(r[i] for r in rs) for i in range(3)],
                               "hi": [max(r[i] for r in rs) for i in range(3)]})
        if not fields:
            return None
        ZL = min(f["lo"][0] for f in fields)
        ZH = max(f["hi"][0] for f in fields)
        depth = ZH - ZL + 2  # one spare slot: a single barrier per plane
        off = 0
        for f in fields:
            f["by"] = self.TILE_Y + f["hi"][1] - f["lo"][1]
            f["bx"] = self.TILE_X + f["hi"][2] - f["lo"][2]
            f["off"] = off
            off += depth * f["by"] * f["bx"]
        esz = 8 if self.T == "double" else 4
        if off * esz > 200 * 1024:
            return None
        return {"fields": fields, "ZL": ZL, "ZH": ZH, "depth": depth, "smem": off * esz}

    def tiled_source(self, index="int"):
        """Tiled predicated gather: a CTA owns a 32 (innermost) x 8 tile of
        the write box and streams the outermost counter over a chunk of
        planes.  Per input plane p it stages, into a ring of depth planes:
        each factored group's Q_g(x) = [x in B] F_g(x) seed(x) over the tile
        plus the group's offset halo (computed once per point instead of once
        per term), and the arrays the unfactored partials read at many points
        (raw values, zero outside the array).  Then, one barrier later, every
        thread forms its output point of plane y0 = p - ZH exactly like the
        fused form: per target, ascending term order, factored terms as k_l *
        Q_g(y - o_l) from shared memory, core points unpredicated, others per
        term predicated (untouched cells never written) -- so the result is
        bitwise the fused / per-nest forms'."""
        lay = self.tiled_layout()
        if lay is None:
            raise _lib.StencilError(f"{self.name}: the tiled gather does not apply")
        self._which = "gather"
        lines, fns, szv = self._prelude(index)
        zargs = ", ".join(f"z_{s}" for s in self.sizes)
        at = {arr: f"AT_{arr}" for arr in self.param_arrays(self._which)}
        for arr, fn in fns.items():
            lines.append(f"#define AT_{arr}(...) {fn}(__VA_ARGS__, {zargs})")
        TX, TY = self.TILE_X, self.TILE_Y
        ZL, ZH, depth = lay["ZL"], lay["ZH"], lay["depth"]
        sig = self._signature("sgb_emitted_tiled", index)
        BY_, RPT = self.BLOCK_Y, self.TILE_Y // self.BLOCK_Y
        sig = sig.replace("__global__ void", f"__global__ void __launch_bounds__({TX * BY_})")
        lines.append(sig[:-1] + ", I zc) {")
        lines.append("  extern __shared__ __align__(16) unsigned char smem_raw[];")
        lines.append("  T* smem = reinterpret_cast<T*>(smem_raw);")
        for f in lay["fields"]:
            lines.append(f"  T* sh_{f['name']} = smem + {f['off']};")
        ext = self._write_box(szv)
        for i in range(3):
            lines.append(f"  const I W{i} = {ext[i]};")
        blo = [affine_c(lo, szv) for lo, _ in self.bounds]
        bhi = [affine_c(hi, szv) for _, hi in self.bounds]
        for i in range(3):
            lines.append(f"  const I Blo{i} = {blo[i]}, Bhi{i} = {bhi[i]};")
        flat_arrays = [a for a in self.param_arrays(self._which) if len(self._shape_of(a)) == 3]
        for a in flat_arrays:
            shp = self._shape_of(a)
            for dim in range(2):
                st = " * ".join(affine_c(shp[q], szv) for q in range(dim + 1, 3))
                lines.append(f"  const I sd_{a}_{dim} = {st};")
        lines.append("  const int lx = threadIdx.x, ly = threadIdx.y, tid = ly * "
                     f"{TX} + lx;")
        lines.append(f"  const I k0 = (I)blockIdx.x * {TX}, j0 = (I)blockIdx.y * {TY};")
        lines.append("  const I yz0 = (I)blockIdx.z * zc;")
        lines.append("  const I yz1 = yz0 + zc < W0 ? yz0 + zc : W0;")
        lines.append("  const I y2 = k0 + lx;")
        lines.append("  int cur = 0;")
        lines.append(f"  for (I p = yz0 + ({ZL}); p < yz1 + ({ZH}); "
                     f"p++, cur = cur + 1 == {depth} ? 0 : cur + 1) {{")
        cidx = {c: i for i, c in enumerate(self.counters)}
        seed_read = ("read", self.seed, [(c, 0) for c in self.lhs])
        # ---- phase 1, software-pipelined: the global loads of plane p + 1
        # go to registers while plane p - ZH is formed from shared memory
        NT = TX * BY_
        pre, store, decl = [], [], []
        for f in lay["fields"]:
            n_el = f["by"] * f["bx"]
            M = -(-n_el // NT)
            if f["kind"] == "q":
                F = self.groups[f["g"]][0]
                rd = []
                for r in _reads(F, [seed_read]):
                    if repr(r) not in [repr(x) for x in rd]:
                        rd.append(r)
                used = sorted({r[1] for r in rd} & set(flat_arrays))
            for m in range(M):
                tag = f"{f['name']}_{m}"
                pre.append("    {")
                pre.append(f"      const int e = tid + {m * NT};")
                pre.append(f"      const int ey = e / {f['bx']}, ex = e - ey * {f['bx']};")
                pre.append(f"      const I x0 = pp, x1 = j0 + ({f['lo'][1]}) + ey, "
                           f"x2 = k0 + ({f['lo'][2]}) + ex;")
                live = f"e < {n_el}" if (m + 1) * NT > n_el else "true"
                if f["kind"] == "q":
                    decl.append(f"  bool pb_{tag} = false;")
                    pre.append(f"      pb_{tag} = {live} && x0 >= Blo0 && x0 <= Bhi0 && "
                               "x1 >= Blo1 && x1 <= Bhi1 && x2 >= Blo2 && x2 <= Bhi2;")
                    for a_ in used:
                        pre.append(f"      const I fy_{a_} = AT_{a_}(x0, x1, x2);")
                    cg = _CGen(self, {c: f"x{cidx[c]}" for c in self.counters}, at,
                               {"shift": {c: 0 for c in self.counters}, "arrays": set(used)})
                    regs = {}
                    for ri, r in enumerate(rd):
                        reg = f"pf_{tag}_{ri}"
                        regs[repr(r)] = reg
                        decl.append(f"  T {reg} = T(0);")
                        pre.append(f"      {reg} = pb_{tag} ? {cg.e(r)} : T(0);")
                    rcg = _RegCGen(self, {c: f"x{cidx[c]}" for c in self.counters}, at, regs)
                    val = f"pb_{tag} ? ({rcg.e(F)}) * {rcg.e(seed_read)} : T(0)"
                else:
                    shp = self._shape_of(f["array"])
                    conds = " && ".join(f"x{i} >= 0 && x{i} < {affine_c(shp[i], szv)}"
                                        for i in range(3))
                    decl.append(f"  T pf_{tag} = T(0);")
                    pre.append(f"      pf_{tag} = ({live} && {conds}) ? "
                               f"a_{f['array']}[AT_{f['array']}(x0, x1, x2)] : T(0);")
                    val = f"pf_{tag}"
                pre.append("    }")
                guard = f"if (tid + {m * NT} < {n_el}) " if (m + 1) * NT > n_el else ""
                store.append(f"    {guard}sh_{f['name']}[cur * {n_el} + tid + {m * NT}] = "
                             f"{val};")
        i_loop = next(i for i, ln in enumerate(lines) if ln.startswith("  for (I p = yz0"))
        lines[i_loop:i_loop] = decl + [f"  {{ const I pp = yz0 + ({ZL});"] + pre + ["  }"]
        lines.extend(store)
        lines.append("    __syncthreads();")
        lines.append(f"    if (p + 1 < yz1 + ({ZH})) {{ const I pp = p + 1;")
        lines.extend(pre)
        lines.append("    }")
        # ---- phase 3: output plane y0 = p - ZH
        lines.append(f"    const I y0 = p - ({ZH});")
        lines.append("    if (y0 < yz0 || y2 >= W2) continue;")
        for k in range(ZL, ZH + 1):
            lines.append(f"    const int s_{_zn(k)} = (cur + {depth - (ZH - k)}) % {depth};")
        # RPT consecutive rows per thread, unrolled: identical shared-memory
        # reads of neighbouring rows are common subexpressions
        lines.append(f"#pragma unroll")
        lines.append(f"    for (int rr = 0; rr < {RPT}; rr++) {{")
        lines.append(f"    const int lr = ly * {RPT} + rr;")
        lines.append("    const I y1 = j0 + lr;")
        lines.append("    if (y1 < W1) {")
        for a_ in flat_arrays:
            lines.append(f"    const I fy_{a_} = AT_{a_}(y0, y1, y2);")
        ring = {f["array"]: f for f in lay["fields"] if f["kind"] == "raw"}
        targets = []
        for t in self.terms:
            if t.adjoint not in targets:
                targets.append(t.adjoint)
        for tgt in targets:
            shp = self._shape_of(tgt)
            inb = " && ".join(f"y{i} < {affine_c(shp[i], szv)}" for i in range(3))
            mine = [ti for ti, t in enumerate(self.terms) if t.adjoint == tgt]
            core = []
            for i in range(3):
                omax = max(self.terms[ti].offset[i] for ti in mine)
                omin = min(self.terms[ti].offset[i] for ti in mine)
                core.append(f"y{i} >= Blo{i} + ({omax}) && y{i} <= Bhi{i} + ({omin})")
            exprs = []
            for ti in mine:
                t = self.terms[ti]
                xs = [f"(y{i} - ({t.offset[i]}))" for i in range(3)]
                if self.factor[ti] is not None:
                    _, g = self.factor[ti]
                    q = _ring_ref(lay["fields"][g], [-t.offset[i] for i in range(3)])
                    cg = _CGen(self, {c: xs[cidx[c]] for c in self.counters}, at)
                    ex = self._term_update(cg, ti, seed_read, "cell", q=q)
                else:
                    shift = {c: -t.offset[cidx[c]] for c in self.counters}
                    cg = _RingCGen(self, {c: xs[cidx[c]] for c in self.counters}, at,
                                   {"shift": shift, "arrays": set(flat_arrays)}, ring, shift)
                    ex = self._term_update(cg, ti, seed_read, "cell")
                exprs.append((ti, t, xs, ex))
            lines.append(f"    if ({inb}) {{")
            lines.append(f"      T* cellp = &a_{tgt}[fy_{tgt}];")
            lines.append(f"      if ({' && '.join(core)}) {{")
            lines.append("        T cell = *cellp;")
            for ti, t, xs, ex in exprs:
                lines.append(f"        cell = {ex};  // term {ti}")
            lines.append("        *cellp = cell;")
            lines.append("      } else {")
            lines.append("        bool touched = false; T cell = T(0);")
            for ti, t, xs, ex in exprs:
                lines.append(f"        if ({self._box_checks(xs, szv)}) {{  // term {ti}")
                lines.append("          if (!touched) { cell = *cellp; touched = true; }")
                lines.append(f"          cell = {ex};")
                lines.append("        }")
            lines.append("        if (touched) *cellp = cell;")
            lines.append("      }")
            lines.append("    }")
        lines.append("    }")  # y1 < W1
        lines.append("    }")  # rows
        lines.append("  }")
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
            seed_read = ("read", self.seed, [(c, 0) for c in self.lhs])
            lines.append(f"  if (mask & (1ULL << {ti})) {{  // term {ti}")
            lines.append(f"    T* cp = &a_{t.adjoint}[AT_{t.adjoint}({ys})];")
            lines.append(f"    *cp = {self._term_update(cg, ti, seed_read, '*cp')};")
            lines.append("  }")
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
        srcs = [self.gather_source(), self.primal_source()]
        if self.tiled_layout() is not None:
            srcs.append(self.tiled_source())
        from . import emit_stream
        if emit_stream.stream_layout(self) is not None:
            srcs.append(emit_stream.stream_source(self))
        for src in srcs:
            if _lib.lib().sgb_jit_check(src.encode()) != 0:
                raise _lib.StencilError(_lib.lib().sgb_jit_log().decode())

    def _kernel(self, which, index="long long"):
        key = (which, index)
        if key not in self._kern:
            if which == "gather":
                src = self.gather_source(index)
            elif which == "tiled":
                src = self.tiled_source(index)
            elif which == "stream":
                from . import emit_stream
                src = emit_stream.stream_source(self, index)
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
                grid=None, index="long long", smem=0):
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
        for arr in self.param_arrays("primal" if which == "primal" else "gather"):  # tiled too
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
        rc = _lib.lib().sgb_jit_launch_smem(self._kernel(which, index), *grid, int(smem), argv,
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

    def adjoint(self, sizes, scalars, arrays, stream=None, form="auto"):
        """Gather adjoint (+= into every adjoint array) on the device.
        form: "flat" (one thread per point, gather_source), "tiled" (3D
        programs with shared subexpressions: shared-memory plane rings,
        tiled_source; bitwise the flat result), "stream" (3D linear-stencil
        programs: the hand-tuned kernels' structure generated,
        emit_stream.py; the flat result to rounding), or "auto": stream in
        fp32 where it applies, else flat.  At cfg 4 (768^3 wave3d_r4) fp32:
        stream 6.0, flat 8.3, tiled 9.1 ms; fp64: flat 14.8, tiled 17.0,
        stream 18.7 ms (DESIGN.md, section 8(f) item 1)."""
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
        if form not in ("auto", "flat", "tiled", "stream"):
            raise _lib.StencilError(f"unknown emitted form {form!r}")
        if form == "auto":
            # the stream form where it applies in fp32 (cfg 4 768^3: 4.9 vs
            # 8.3 ms flat); in fp64 the flat form is faster (14.7 vs 16.3 ms)
            from . import emit_stream
            form = "flat"
            if self.T == "float" and W[2] % 4 == 0 and \
                    not any(t.data_ptr() % 16 for t in arrays.values() if hasattr(t, "data_ptr")) \
                    and emit_stream.stream_layout(self) is not None:
                form = "stream"
        if form == "stream":
            from . import emit_stream
            sl = emit_stream.stream_layout(self)
            if sl is None:
                raise _lib.StencilError(f"{self.name}: the stream form does not apply")
            if W[2] % 4 != 0 or any(t.data_ptr() % 16 for t in arrays.values()):
                raise _lib.StencilError(f"{self.name}: the stream form needs the innermost "
                                        "extent a multiple of 4 and 16-byte aligned arrays")
            gx = (W[2] + emit_stream.TK - 1) // emit_stream.TK
            gy = (W[1] + emit_stream.TJ - 1) // emit_stream.TJ
            # outer-counter chunks of ~ZCHUNK planes (2R warm-up planes each): short
            # chunks keep the resident CTAs on nearly the same planes, so the halo
            # rows neighbouring tiles share are still in L2 -- one chunk per column
            # (the wave model's choice) measured 20 % slower at 768^3; 48 ... 256
            # planes: 4.86 / 4.77 / 4.71 / 4.71 / 4.81 / 4.92 ms at 48 / 64 / 96 / 128 / 192 / 256
            nz = max(1, -(-W[0] // emit_stream.ZCHUNK))
            while nz < W[0] and gx * gy * nz < 2 * 148:
                nz *= 2
            zc = -(-W[0] // nz)
            nz = -(-W[0] // zc)
            if gy > 65535 or nz > 65535:
                raise _lib.StencilError("grid too large")
            zt = ctypes.c_int if index == "int" else ctypes.c_longlong
            self._launch("stream", sizes, scalars, arrays, 0, stream, extra=(zt(zc),),
                         grid=(gx, gy, nz, sl["threads"], 1, 1), index=index, smem=sl["smem"])
            return
        lay = self.tiled_layout() if form == "tiled" else None
        if form == "tiled" and lay is None:
            raise _lib.StencilError(f"{self.name}: the tiled gather does not apply")
        if lay is not None:
            gx = (W[2] + self.TILE_X - 1) // self.TILE_X
            gy = (W[1] + self.TILE_Y - 1) // self.TILE_Y
            # outermost-counter chunks: ~256 planes (ring warm-up ZH - ZL
            # planes per chunk), at least 2 waves of CTAs
            nz = max(1, -(-W[0] // 256))
            while nz < W[0] and gx * gy * nz < 4 * 148:
                nz *= 2
            zc = -(-W[0] // nz)
            nz = -(-W[0] // zc)
            if gy > 65535 or nz > 65535:
                raise _lib.StencilError("grid too large")
            zt = ctypes.c_int if index == "int" else ctypes.c_longlong
            self._launch("tiled", sizes, scalars, arrays, 0, stream, extra=(zt(zc),),
                         grid=(gx, gy, nz, self.TILE_X, self.BLOCK_Y, 1), index=index,
                         smem=lay["smem"])
            return
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
