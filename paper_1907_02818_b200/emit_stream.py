"""Streaming form of the emitted gather (3D): the hand-tuned radius-4 kernel's
structure, generated from the program.

A CTA owns a 32 (innermost counter) x 16 tile and streams the outermost
counter over a chunk of planes.  The program's terms are sorted into

* rings: per target, either its factored terms (k_l * Q_g(y - o_l), the
  shared subexpressions of EmittedProblem._factorise) or ONE term whose
  partial is (pointwise factors) x (a linear combination of shifted reads of
  one array A) -- the c_b term of the wave stencils, whose partial holds the
  Laplacian of u_1;
* pointwise terms: partials that read only at the output point.

Per plane the CTA stages every field a ring reads in shared memory with
cp.async (16-byte copies, zero-filled off the grid; nothing is held in
registers while in flight): the raw arrays of the taps straight into 4-plane
rings, the arrays Q_g = [x in B] F_g(x) seed(x) is formed from into per-thread
staging slots; planes p + 1 and p + 2 are in flight while plane p is
consumed, one commit group per plane and one barrier per plane.  The
copying thread forms Q_g for its own elements (double-buffered plane), then
one role of threads per target-with-a-ring forms, for RPT rows x 4
consecutive points each, the taps of its ring with outer offset di from k
windows held in registers and adds them into the register-ring slot of
output plane p - di.  The emit's own reads (the old adjoint values, the
pointwise arrays at the output point) ride in the same cp.async groups,
requested with the plane that completes their output plane (fp32; when the
slots would leave one CTA per SM they are loaded at the start of the taps).
Tiles whose staged box lies inside the primal box take a copy of the staging
code with CTA-uniform predicates only.
Plane p - R is complete: its owner writes old value + ring (or
pointwise factors x ring x seed) + the pointwise terms, predicated per point
off the core box (untouched cells are never written).  The sums run in a
different order than the flat form's per-cell term order, so the results
agree with it -- and with the reference's run_program -- to floating-point
rounding, not bit for bit.

Applies when: 3D; every array has the write box's shape; the seed and the
non-factored terms sit at the output point (offset 0, centred partials);
factored subexpressions F_g read only at their point; every tap |dk| <= 4;
at most one ring per target and at most two rings.  The launcher also needs
the innermost extent to be a multiple of 4 and 16-byte aligned arrays.
"""
from __future__ import annotations

from .emitter import _CGen, _RegCGen, _reads, affine_c

TK, TJ, HK = 32, 16, 4  # tile: 32 innermost x 16 rows (32 rows: 6.02 vs 5.90 ms at cfg 4); k halo
KQ = TK // 4            # k quads per row
RPT = 1                 # rows per thread (2: rows shared in registers, but 224 registers
                        # and 8 warps per SM; 1: ~128 registers, 16 warps per SM)


ZCHUNK = 128            # planes of the outer counter per CTA (launcher)
L2HINT = ""             # cp.async L2 prefetch qualifier ("", ".L2::128B", ".L2::256B")
NSTG = 4                # planes of a staged field in shared memory (cp.async ring)
PD = 2                  # planes requested ahead of the one being consumed
UNROLL = False          # plane loop unrolled by the ring size (static modular slots, no
                        # shift-register moves; a RING-times larger body)


def _role(rpt):
    return KQ * (TJ // rpt)  # threads per ring role
BWQ = (TK + 2 * HK) // 4  # 4-element groups per staged row (10)


def _centred(node):
    return all(all(o == 0 for _, o in r[2]) for r in _reads(node, []))


def _linear_form(ep, node):
    """node = sum of +-c_e * A[x + e] (one array A, counter-aligned reads,
    c_e free of reads) -> (A, [(e, coef node, sign)]) else None."""
    out = []

    def walk(n, sign):
        k = n[0]
        if k in ("add", "sub"):
            return walk(n[1], sign) and walk(n[2], sign if k == "add" else -sign)
        if k == "neg":
            return walk(n[1], -sign)
        if k == "read":
            out.append((n, ("num", "1"), sign))
            return True
        if k == "mul":
            a, b = n[1], n[2]
            if b[0] == "read" and not _reads(a, []):
                out.append((b, a, sign))
                return True
            if a[0] == "read" and not _reads(b, []):
                out.append((a, b, sign))
                return True
        return False
    if not walk(node, 1) or len(out) < 2:
        return None
    arrays = {r[1] for r, _, _ in out}
    if len(arrays) != 1:
        return None
    A = arrays.pop()
    taps = []
    for r, coef, sign in out:
        if [c for c, _ in r[2]] != ep.counters:
            return None
        taps.append((tuple(o for _, o in r[2]), coef, sign))
    return A, taps


def stream_layout(ep):
    """The form's rings, fields and roles, or None when it does not apply."""
    if ep.d != 3 or not ep.terms or list(ep.lhs) != ep.counters:
        return None
    box = ep._shape_of(ep.terms[0].adjoint)
    for a in ep.param_arrays("gather"):
        if ep._shape_of(a) != box:
            return None
    targets = []
    for t in ep.terms:
        if t.adjoint not in targets:
            targets.append(t.adjoint)
    rings = {}   # target -> {"kind": "fac"|"lin", "taps": [(field, (di,dj,dk), coef, sign)], ...}
    points = {T: [] for T in targets}
    for ti, t in enumerate(ep.terms):
        o = tuple(t.offset)
        T = t.adjoint
        if ep.factor[ti] is not None:
            k, g = ep.factor[ti]
            if not _centred(ep.groups[g][0]):
                return None
            r = rings.setdefault(T, {"kind": "fac", "taps": [], "terms": []})
            if r["kind"] != "fac":
                return None
            r["taps"].append((f"q{g}", tuple(-x for x in o), k, 1))
            r["terms"].append(ti)
            continue
        if any(o):
            return None
        part = ep.partials[ti]
        if _centred(part):
            points[T].append(ti)
            continue
        chain, n = [], part
        while n[0] == "mul":
            chain.insert(0, n[2])
            n = n[1]
        chain.insert(0, n)
        lin = [i for i, f in enumerate(chain) if not _centred(f)]
        if len(lin) != 1 or T in rings:
            return None
        lf = _linear_form(ep, chain[lin[0]])
        if lf is None:
            return None
        A, taps = lf
        rings[T] = {"kind": "lin", "taps": [(f"r_{A}", e, c, s) for e, c, s in taps],
                    "terms": [ti], "chain": chain, "li": lin[0]}
    roles = [T for T in targets if T in rings]
    if not roles or len(roles) > 2:
        return None
    taps = [tp for T in roles for _, tp, _, _ in rings[T]["taps"]]
    if any(abs(tp[2]) > HK for tp in taps):
        return None
    HJ = max(abs(tp[1]) for tp in taps)
    Rm = max(abs(tp[0]) for tp in taps)
    if HJ > 8 or Rm > 8:
        return None
    fields = {}
    for T in roles:
        for f, _, _, _ in rings[T]["taps"]:
            if f not in fields:
                fields[f] = {"kind": "q", "g": int(f[1:])} if f.startswith("q") else \
                    {"kind": "raw", "array": f[2:]}
    BJ = TJ + 2 * HJ
    esz = 8 if ep.T == "double" else 4
    seed_read = ("read", ep.seed, [(c, 0) for c in ep.lhs])
    off = 0
    for f in fields.values():
        f["off"] = off
        if f["kind"] == "q":
            # the formed Q plane, double-buffered, + an NSTG-plane cp.async ring
            # per array F_g and the seed read (consumed by the copying thread)
            off += 2 * BJ * BWQ * 4
            rd = []
            for r in _reads(ep.groups[f["g"]][0], [seed_read]):
                if r[1] not in rd:
                    rd.append(r[1])
            f["reads"], f["st_off"] = rd, off
            off += len(rd) * NSTG * BJ * BWQ * 4
        else:
            off += NSTG * BJ * BWQ * 4  # the raw planes themselves, read by the taps
    lay = {"rings": rings, "points": points, "roles": roles, "targets": targets,
           "fields": fields, "HJ": HJ, "R": Rm, "RING": 2 * Rm + 1, "BJ": BJ,
           "rpt": RPT, "unroll": UNROLL, "threads": _role(RPT) * len(roles)}
    # the emit's own reads (old adjoint values, pointwise arrays at the output
    # point) go through per-thread cp.async slots too: [slot][row][thread of the
    # role][4], requested with the plane that completes them
    lay["emit"] = {}
    eoff = off
    for ri, T in enumerate(roles):
        mine = [(T, True)] + ([(T2, False) for T2 in targets if T2 not in rings]
                              if ri == 0 else [])
        for Tt, rg in mine:
            for a in _target_reads(ep, lay, Tt, rg):
                lay["emit"][(Tt, a)] = eoff
                eoff += NSTG * RPT * _role(RPT) * 4
    # ... when two CTAs per SM still fit (fp32 at cfg 4: 101 KB per CTA; in fp64
    # the slots would leave one CTA per SM -- 16.4 -> 19 ms -- so the emit then
    # loads its values from global memory at the start of the plane's taps)
    per_sm = max(1, 512 // lay["threads"])  # CTAs per SM the launch bounds ask for
    lay["emit_async"] = eoff * esz <= (227 // per_sm - 1) * 1024
    if lay["emit_async"]:
        off = eoff
    lay["smem"] = off * esz
    if lay["smem"] > 227 * 1024:  # does not fit one CTA's shared memory
        return None
    return lay


def stream_source(ep, index="int"):
    lay = stream_layout(ep)
    if lay is None:
        raise ValueError(f"{ep.name}: the stream form does not apply")
    ep._which = "gather"
    lines, fns, szv = ep._prelude(index)
    zargs = ", ".join(f"z_{s}" for s in ep.sizes)
    at = {arr: f"AT_{arr}" for arr in ep.param_arrays("gather")}
    for arr, fn in fns.items():
        lines.append(f"#define AT_{arr}(...) {fn}(__VA_ARGS__, {zargs})")
    dbl = ep.T == "double"
    # 4 consecutive elements through 16-byte accesses
    if dbl:
        lines += ["__device__ __forceinline__ void ld4(const T* p, T* o) {",
                  "  const double2 a = *reinterpret_cast<const double2*>(p);",
                  "  const double2 b = *reinterpret_cast<const double2*>(p + 2);",
                  "  o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y; }",
                  "__device__ __forceinline__ void st4(T* p, const T* v) {",
                  "  *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);",
                  "  *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]); }"]
    else:
        lines += ["__device__ __forceinline__ void ld4(const T* p, T* o) {",
                  "  const float4 a = *reinterpret_cast<const float4*>(p);",
                  "  o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = a.w; }",
                  "__device__ __forceinline__ void st4(T* p, const T* v) {",
                  "  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]); }"]
    # 4 consecutive elements global -> shared without registers (zero-filled
    # when `ok` is false); groups are committed once per plane
    lines += ["__device__ __forceinline__ void cpa4(unsigned d, const T* src, bool ok) {",
              "  const int nb = ok ? 16 : 0;"]
    for half in range(2 if dbl else 1):
        lines += [f'  asm volatile("cp.async.cg.shared.global{L2HINT} [%0], [%1], 16, %2;" :: '
                  f'"r"(d + {16 * half}), "l"(reinterpret_cast<const char*>(src) + '
                  f'{16 * half}), "r"(nb) : "memory");']
    lines += ["}",
              "__device__ __forceinline__ void cpa_commit() {",
              '  asm volatile("cp.async.commit_group;" ::: "memory"); }',
              "template <int N> __device__ __forceinline__ void cpa_wait() {",
              '  asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }']
    for T in lay["roles"]:
        if lay["rings"][T]["kind"] == "fac":
            lines += _reach_fn(ep, lay, T, index)
    Rm, RING, HJ, BJ = lay["R"], lay["RING"], lay["HJ"], lay["BJ"]
    rpt = lay["rpt"]
    NTH = lay["threads"]
    fields, rings, roles = lay["fields"], lay["rings"], lay["roles"]
    seed_read = ("read", ep.seed, [(c, 0) for c in ep.lhs])
    sig = ep._signature("sgb_emitted_stream", index)
    # at most 128 registers per thread: 16 warps per SM in one or more CTAs
    sig = sig.replace("__global__ void",
                      f"__global__ void __launch_bounds__({NTH}, {max(1, 512 // NTH)})")
    L = lines
    L.append(sig[:-1] + ", I zc) {")
    L.append("  extern __shared__ __align__(16) unsigned char smem_raw[];")
    L.append("  T* smem = reinterpret_cast<T*>(smem_raw);")
    for name, f in fields.items():
        L.append(f"  T* sh_{name} = smem + {f['off']};")
        if f["kind"] == "q":
            L.append(f"  T* st_{name} = smem + {f['st_off']};")
    ext = ep._write_box(szv)
    for i in range(3):
        L.append(f"  const I W{i} = {ext[i]};")
    for i, (lo, hi) in enumerate(ep.bounds):
        L.append(f"  const I Blo{i} = {affine_c(lo, szv)}, Bhi{i} = {affine_c(hi, szv)};")
    L.append("  const I sd1 = W2, sd0 = W1 * W2;")
    ROLE = _role(rpt)
    L.append(f"  const int tid = threadIdx.x, role = tid / {ROLE}, rt = tid - role * {ROLE};")
    L.append(f"  const int tx = rt % {KQ}, ty = rt / {KQ};")
    L.append(f"  const I k0 = (I)blockIdx.x * {TK}, j0 = (I)blockIdx.y * {TJ};")
    L.append("  const I yz0 = (I)blockIdx.z * zc;")
    L.append("  const I yz1 = yz0 + zc < W0 ? yz0 + zc : W0;")
    L.append(f"  const I kc = k0 + 4 * tx, jr = j0 + {rpt} * ty;")
    L.append(f"  const I pstart = yz0 - ({Rm}), pend = yz1 + ({Rm});")
    # ---- staging: `pre` requests plane pp into ring slot ps with cp.async (no
    # registers held across the planes in flight); `store` forms the Q planes
    # from the copying thread's own staged elements (registers -> smem)
    NE = BJ * BWQ
    M = -(-NE // NTH)
    EB = 8 if dbl else 4  # element bytes
    pre, store, decl = [], [], []
    decl.append("  const unsigned smem_u = (unsigned)__cvta_generic_to_shared(smem);")
    decl.append("  const I sdp = W1 * W2;")
    # per thread and staged element group: everything that does not depend on
    # the plane (row / column, in-grid and in-box tests, the in-plane offset)
    for m in range(M):
        decl.append(f"  const int se{m} = tid + {m * NTH};")
        decl.append(f"  const int srow{m} = se{m} / {BWQ}, sc4{m} = se{m} - srow{m} * {BWQ};")
        decl.append(f"  const I sx1{m} = j0 - {HJ} + srow{m}, sx2{m} = k0 - {HK} + 4 * sc4{m};")
        decl.append(f"  const bool sin{m} = se{m} < {NE} && sx1{m} >= 0 && sx1{m} < W1 && "
                    f"sx2{m} >= 0 && sx2{m} < W2;")
        decl.append(f"  const I soff{m} = sin{m} ? sx1{m} * W2 + sx2{m} : (I)0;")
        decl.append(f"  unsigned spm{m} = 0u;  // lanes of the group inside the box (rows too)")
        decl.append(f"  if (sin{m} && sx1{m} >= Blo1 && sx1{m} <= Bhi1)")
        decl.append("    for (int l = 0; l < 4; l++)")
        decl.append(f"      if (sx2{m} + l >= Blo2 && sx2{m} + l <= Bhi2) spm{m} |= 1u << l;")
    # A tile whose staged box lies inside the primal box in the inner two
    # counters (the interior of the grid) needs none of the per-thread tests:
    # `tin` picks a second copy of the staging code with CTA-uniform predicates
    # only (the plane tests).  Same values either way.
    decl.append(f"  const bool tin = j0 - {HJ} >= Blo1 && j0 + {TJ + HJ - 1} <= Bhi1 && "
                f"k0 - {HK} >= Blo2 && k0 + {TK + HK - 1} <= Bhi2 && Blo1 >= 0 && Bhi1 < W1 && "
                "Blo2 >= 0 && Bhi2 < W2;")

    def staging(fast):
        pre, store = [], []
        pre.append("    const bool pokr = pp >= 0 && pp < W0, pokq = pokr && pp >= Blo0 && "
                   "pp <= Bhi0;")
        store.append("      const bool pin = p >= Blo0 && p <= Bhi0 && p >= 0 && p < W0;")
        for name, f in fields.items():
            if f["kind"] == "q":
                F = ep.groups[f["g"]][0]
                rd = f["reads"]
            for m in range(M):
                guard = f"if (se{m} < {NE}) " if (m + 1) * NTH > NE else ""
                pre.append(f"    {guard}{{")
                if f["kind"] == "q":
                    # off the box in the outer counter, or the whole group off it
                    # in the inner two: Q = 0 whatever is read -- nothing is
                    pre.append("      const bool ok = pokq" + ("" if fast else f" && spm{m} != 0u")
                               + ";")
                else:
                    pre.append("      const bool ok = pokr" + ("" if fast else f" && sin{m}") + ";")
                pre.append(f"      const I fx = ok ? pp * sdp + soff{m} : (I)0;")
                if f["kind"] == "q":
                    for ri, arr in enumerate(rd):
                        pre.append(f"      cpa4(smem_u + ({f['st_off']} + ({ri * NSTG} + ps) * "
                                   f"{NE * 4} + se{m} * 4) * {EB}, a_{arr} + fx, ok);")
                else:
                    pre.append(f"      cpa4(smem_u + ({f['off']} + ps * {NE * 4} + se{m} * 4) * "
                               f"{EB}, a_{f['array']} + fx, ok);")
                pre.append("    }")
                if f["kind"] != "q":
                    continue
                store.append(f"      {guard}{{")
                store.append("        const unsigned pm = pin ? " + ("15u" if fast else f"spm{m}")
                             + " : 0u;")
                for ri, arr in enumerate(rd):
                    store.append(f"        T pf_{ri}[4]; ld4(st_{name} + ({ri * NSTG} + rs) * "
                                 f"{NE * 4} + se{m} * 4, pf_{ri});")
                vals = []
                for lane in range(4):
                    regs = {}
                    for r in _reads(F, [seed_read]):
                        regs[repr(r)] = f"pf_{rd.index(r[1])}[{lane}]"
                    rcg = _RegCGen(ep, {}, at, regs)
                    vals.append(f"((pm >> {lane}) & 1u) ? ({rcg.e(F)}) * {rcg.e(seed_read)} : "
                                "T(0)")
                store.append(f"        const T v_[4] = {{{', '.join(vals)}}};")
                store.append(f"        st4(sh_{name} + bsel * {NE * 4} + se{m} * 4, v_);")
                store.append("      }")
        # the emit's reads for output plane pp - R ride in plane pp's group
        pre.append(f"    {{ const I yq = pp - ({Rm}); const bool eq_ok = yq >= yz0 && yq < yz1"
                   + ("" if fast else " && kc < W2") + ";")
        for ri, T in enumerate(roles):
            pre.append(f"      {'if' if ri == 0 else 'else if'} (role == {ri}) {{")
            mine_q = [(T, True)] + ([(T2, False) for T2 in lay["targets"] if T2 not in rings]
                                    if ri == 0 else [])
            for Tt, rg in mine_q:
                pre += _emit_target(ep, lay, Tt, at, seed_read, ring=rg,
                                    part="request_fast" if fast else "request", rpt=rpt)
            pre.append("      }")
        pre.append("    }")
        return pre, store

    pre_g, store_g = staging(False)
    pre_f, store_f = staging(True)
    pre = ["    if (tin) {"] + ["  " + x for x in pre_f] + ["    } else {"] + \
        ["  " + x for x in pre_g] + ["    }"]
    store = ["      if (tin) {"] + ["  " + x for x in store_f] + ["      } else {"] + \
        ["  " + x for x in store_g] + ["      }"]
    L += decl
    # acc[s] holds output plane p - R + s (a shift register: plane p's taps
    # with outer offset di go to s = R - di; after the emit of acc[0] the
    # ring moves down one slot), so the plane loop is one copy of the code
    L.append(f"  T acc[{RING}][{rpt}][4];")
    L.append("#pragma unroll")
    L.append(f"  for (int q = 0; q < {RING}; q++)")
    L.append("#pragma unroll")
    L.append(f"    for (int h = 0; h < {rpt}; h++)")
    L.append("#pragma unroll")
    L.append("      for (int l = 0; l < 4; l++) acc[q][h][l] = T(0);")
    for d_ in range(PD):  # planes pstart .. pstart + PD - 1 requested up front
        L.append(f"  {{ const I pp = pstart + {d_}; const int ps = {d_ % NSTG};")
        L.append("    if (pp < pend) {")
        L += pre
        L.append("    }")
        L.append("    cpa_commit();")
        L.append("  }")
    L.append("  int bsel = 0, rs = 0;  // rs: ring slot of plane p")
    unroll = lay["unroll"]
    if unroll:
        L.append(f"  for (I base = pstart; base < pend; base += {RING}) {{")
        L.append("#pragma unroll")
        L.append(f"  for (int ph = 0; ph < {RING}; ph++) {{")
        L.append("    const I p = base + ph;")
        L.append("    if (p < pend) {")
    else:
        L.append("#pragma unroll 1")
        L.append("  for (I p = pstart; p < pend; p++) {")
        L.append("    {")
    # plane p has landed (this thread's copies; the others' by the barrier);
    # plane p + PD goes to a slot last read PD + 1 < NSTG + 1 planes ago -- a
    # thread still in plane p - 1's taps reads slot rs - 1, never this one
    L.append(f"      cpa_wait<{PD - 1}>();")
    L.append(f"      {{ const I pp = p + {PD}; const int ps = (rs + {PD}) % {NSTG};")
    L.append("        if (pp < pend) {")
    L += ["    " + x for x in pre]
    L.append("        }")
    L.append("        cpa_commit();")
    L.append("      }")
    L += store
    L.append("      __syncthreads();")
    cg0 = _CGen(ep, {}, at)

    def ring_code(T):
        out = []
        r = rings[T]
        wins = {}
        for fname, tap, _, _ in r["taps"]:
            key = (fname, tap[1])
            wins[key] = wins.get(key, False) or tap[2] != 0
        loaded = set()
        for fname, tap, coef, sgn in r["taps"]:  # tap order = term order
            key = (fname, tap[1])
            for h in range(rpt):
                w = f"w_{fname}_{tap[1] + 8}_{h}"
                if (key, h) not in loaded:
                    loaded.add((key, h))
                    sel = "bsel" if fields[fname]["kind"] == "q" else "rs"
                    base_ = (f"sh_{fname} + {sel} * {NE * 4} + ({rpt} * ty + {h} + "
                             f"{tap[1] + HJ}) * {BWQ * 4} + 4 * tx")
                    if wins[key]:
                        out.append(f"      T {w}[12]; ld4({base_}, {w}); ld4({base_} + 4, {w} + 4);"
                                   f" ld4({base_} + 8, {w} + 8);")
                    else:
                        out.append(f"      T {w}[12]; ld4({base_} + 4, {w} + 4);")
            slot = f"(ph + {(-tap[0]) % RING}) % {RING}" if unroll else Rm - tap[0]
            c = cg0.e(coef if coef is not None else ("num", "1"))
            c = f"-({c})" if sgn < 0 else f"({c})"
            for h in range(rpt):
                for lane in range(4):
                    a_ = f"acc[{slot}][{h}][{lane}]"
                    v = f"w_{fname}_{tap[1] + 8}_{h}[{4 + lane + tap[2]}]"
                    out.append(f"      {a_} = fma({c}, {v}, {a_});" if ep.fma else
                               f"      {a_} = {a_} + {c} * {v};")
        return out

    # ---- per role: the emitted plane's global values requested first (their
    # latency hides behind the taps), the taps of plane p, then output plane
    # y0 = p - R
    L.append(f"      const I y0 = p - ({Rm});")
    L.append("      const bool emit_ok = y0 >= yz0 && y0 < yz1 && kc < W2;")
    L.append(f"      const int es = {'(ph + ' + str((-Rm) % RING) + ') % ' + str(RING) if unroll else '0'};")
    pointwise_only = [T for T in lay["targets"] if T not in rings]
    for ri, T in enumerate(roles):
        L.append(f"      {'if' if ri == 0 else 'else if'} (role == {ri}) {{")
        mine_t = [(T, True)] + ([(T2, False) for T2 in pointwise_only] if ri == 0 else [])
        for Tt, rg in mine_t:
            L += _emit_target(ep, lay, Tt, at, seed_read, ring=rg, part="load", rpt=rpt)
        L += ring_code(T)
        L.append("      if (emit_ok) {")
        for Tt, rg in mine_t:
            L += _emit_target(ep, lay, Tt, at, seed_read, ring=rg, part="compute", rpt=rpt)
        L.append("      }")
        L.append("      }")
    if unroll:  # the emitted slot is reused for output plane y0 + RING
        L.append("#pragma unroll")
        L.append(f"      for (int h = 0; h < {rpt}; h++)")
        L.append("#pragma unroll")
        L.append("        for (int l = 0; l < 4; l++) acc[es][h][l] = T(0);")
    else:
        L.append("#pragma unroll")
        L.append(f"      for (int q = 0; q + 1 < {RING}; q++)")
        L.append("#pragma unroll")
        L.append(f"        for (int h = 0; h < {rpt}; h++)")
        L.append("#pragma unroll")
        L.append("          for (int l = 0; l < 4; l++) acc[q][h][l] = acc[q + 1][h][l];")
        L.append("#pragma unroll")
        L.append(f"      for (int h = 0; h < {rpt}; h++)")
        L.append("#pragma unroll")
        L.append(f"        for (int l = 0; l < 4; l++) acc[{RING - 1}][h][l] = T(0);")
    L.append("      bsel ^= 1;")
    L.append(f"      rs = (rs + 1) % {NSTG};")
    L.append("    }")
    L.append("  }")
    if unroll:
        L.append("  }")
    L.append("}")
    return "\n".join(L) + "\n"


def _reach_fn(ep, lay, T, index):
    """__device__ helper: does any factored term of T reach y (y - o_l in B)?
    A loop over a static offset table, so the frame path stays small."""
    tis = lay["rings"][T]["terms"]
    offs = ", ".join(f"{{{o[0]}, {o[1]}, {o[2]}}}" for o in (ep.terms[ti].offset for ti in tis))
    return [f"__device__ __noinline__ bool fac_reach_{T}({index} y0, {index} y1, {index} y2, "
            f"{index} b0, {index} e0, {index} b1, {index} e1, {index} b2, {index} e2) {{",
            f"  const int off[{len(tis)}][3] = {{{offs}}};",
            f"  for (int l = 0; l < {len(tis)}; l++)",
            "    if (y0 - off[l][0] >= b0 && y0 - off[l][0] <= e0 && y1 - off[l][1] >= b1 &&",
            "        y1 - off[l][1] <= e1 && y2 - off[l][2] >= b2 && y2 - off[l][2] <= e2)",
            "      return true;",
            "  return false;",
            "}"]


def _target_reads(ep, lay, T, ring):
    """Arrays the emit of target T reads at the output point (the pointwise
    partials, the seed, a linear ring's pointwise factors), then T itself."""
    seed_read = ("read", ep.seed, [(c, 0) for c in ep.lhs])
    r = lay["rings"].get(T) if ring else None
    nodes = [ep.partials[ti] for ti in lay["points"][T]] + [seed_read]
    if r and r["kind"] == "lin":
        nodes += [f for i, f in enumerate(r["chain"]) if i != r["li"]]
    reads = []
    for nd in nodes:
        for rd in _reads(nd, []):
            if rd[1] not in reads:
                reads.append(rd[1])
    return reads + [T]


def _emit_target(ep, lay, T, at, seed_read, ring, part, rpt):
    """Emit code of target T for the thread's 2 rows x 4 points: part "load"
    requests the old values and the pointwise arrays at the output point
    into registers, part "compute" forms and stores the results."""
    out = []
    cidx = {c: i for i, c in enumerate(ep.counters)}
    mine = [ti for ti, t in enumerate(ep.terms) if t.adjoint == T]
    r = lay["rings"].get(T) if ring else None
    ring_terms = r["terms"] if r else []
    pts = lay["points"][T]
    # arrays read at the output point by the pointwise parts (vector loads)
    reads = []
    nodes = [ep.partials[ti] for ti in pts] + [seed_read]
    if r and r["kind"] == "lin":
        nodes += [f for i, f in enumerate(r["chain"]) if i != r["li"]]
    for nd in nodes:
        for rd in _reads(nd, []):
            if rd[1] not in reads:
                reads.append(rd[1])
    core = []
    for i in range(3):
        omax = max(ep.terms[ti].offset[i] for ti in mine)
        omin = min(ep.terms[ti].offset[i] for ti in mine)
        lo_, hi_ = ("y0", "y0") if i == 0 else (("y1", "y1") if i == 1 else ("kc", "kc + 3"))
        core.append(f"{lo_} >= Blo{i} + ({omax}) && {hi_} <= Bhi{i} + ({omin})")
    ROLE = _role(rpt)
    if part in ("request", "request_fast"):  # plane pp's group: what output plane pp - R needs
        if not lay["emit_async"]:
            return out
        EB = 8 if ep.T == "double" else 4
        for h in range(rpt):
            out.append("        { const bool ok = eq_ok" +
                       ("" if part == "request_fast" else f" && jr + {h} < W1") + ";")
            out.append(f"          const I fy = ok ? yq * sdp + (jr + {h}) * W2 + kc : (I)0;")
            for a in reads + [T]:
                out.append(f"          cpa4(smem_u + ({lay['emit'][(T, a)]} + ((ps * {rpt} + {h}) * "
                           f"{ROLE} + rt) * 4) * {EB}, a_{a} + fy, ok);")
            out.append("        }")
        return out
    if part == "load" and lay["emit_async"]:
        for h in range(rpt):
            for a in reads + [T]:
                out.append(f"      T e_{T}_{a}_{h}[4]; ld4(smem + {lay['emit'][(T, a)]} + "
                           f"((rs * {rpt} + {h}) * {ROLE} + rt) * 4, e_{T}_{a}_{h});")
        return out
    if part == "load":
        for h in range(rpt):
            for a in reads + [T]:
                out.append(f"      T e_{T}_{a}_{h}[4];")
            out.append(f"      if (emit_ok && jr + {h} < W1) {{")
            out.append(f"        const I fy = (y0 * W1 + jr + {h}) * W2 + kc;")
            for a in reads + [T]:
                out.append(f"        ld4(a_{a} + fy, e_{T}_{a}_{h});")
            out.append("      }")
        return out
    for h in range(rpt):
        out.append(f"        {{ const I y1 = jr + {h};")
        out.append("        if (y1 < W1) {")
        out.append("          const I fy = (y0 * W1 + y1) * W2 + kc;")
        for a in reads:
            out.append(f"          T* v_{a} = e_{T}_{a}_{h};")
        out.append(f"          T* cell = e_{T}_{T}_{h};")
        lane_ex = []
        for lane in range(4):
            regs = {}
            for nd in nodes:
                for rd in _reads(nd, []):
                    regs[repr(rd)] = f"v_{rd[1]}[{lane}]"
            rcg = _RegCGen(ep, {}, at, regs)
            exs = []  # (ti, validity over the 4 lanes' coordinate, update expression)
            if r and r["kind"] == "fac":
                exs.append(("fac", f"cell[{lane}] + acc[es][{h}][{lane}]"))
            if r and r["kind"] == "lin":
                ti = r["terms"][0]
                prod = None
                for i, f in enumerate(r["chain"]):
                    v = f"acc[es][{h}][{lane}]" if i == r["li"] else f"({rcg.e(f)})"
                    prod = v if prod is None else f"({prod} * {v})"
                S = rcg.e(seed_read)
                exs.append((ti, f"fma({prod}, {S}, cell[{lane}])" if ep.fma else
                            f"cell[{lane}] + {prod} * {S}"))
            for ti in pts:
                P = rcg.e(ep.partials[ti])
                S = rcg.e(seed_read)
                exs.append((ti, f"fma(({P}), {S}, cell[{lane}])" if ep.fma else
                            f"cell[{lane}] + ({P}) * {S}"))
            lane_ex.append(exs)
        out.append(f"          if ({' && '.join(core)}) {{")
        for lane in range(4):
            for _, ex in lane_ex[lane]:
                out.append(f"            cell[{lane}] = {ex};")
        out.append(f"            st4(a_{T} + fy, cell);")
        out.append("          } else {")
        for lane in range(4):
            out.append("            {")
            out.append(f"              const I y2 = kc + {lane}; bool touched = false;")
            for key, ex in lane_ex[lane]:
                if key == "fac":
                    cond = f"fac_reach_{T}(y0, y1, y2, Blo0, Bhi0, Blo1, Bhi1, Blo2, Bhi2)"
                else:
                    cond = ep._box_checks(["y0", "y1", "y2"], {s: f"z_{s}" for s in ep.sizes})
                out.append(f"              if ({cond}) {{ touched = true; cell[{lane}] = {ex}; }}")
            out.append(f"              if (touched) a_{T}[fy + {lane}] = cell[{lane}];")
            out.append("            }")
        out.append("          }")
        out.append("        }")
        out.append("        }")
    return out
