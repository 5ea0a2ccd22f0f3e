/* sg_oracle.c — CPU restatement of the reference adjoint-stencil path.
 *
 * TEST INFRASTRUCTURE ONLY (see sg_oracle.h).  Each function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 * Parity of this restatement is pinned by tests/test_oracle_pins.py against
 * the reference's known-answer tests and against golden vectors produced by
 * the unmodified reference library (tests/golden/, oracle/ref/).
 */
#include "sg_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* 8th-order second-derivative weights as the 17-digit literals of
 * oracle/specs/wave3d_r4.json; the centre coefficient is the value the
 * reference's simplify folds 3*w0 to (symdiff.cpp:44-83). */
static const double W4[5] = {-2.8472222222222223, 1.6, -0.2, 0.025396825396825397,
                             -0.0017857142857142857};
static const double W4_CENTER3 = -8.541666666666668;

static sg_family FAMS[SG_NUM_FAMILIES];
static int fams_ready = 0;

static void set_terms_star(sg_family* f, int arr, int radius, int start) {
  /* all star offsets of the given radius in lexicographic (outer-first)
   * order, which is the active_reads order for one array (symdiff.cpp:204-223) */
  int t = start;
  int d = f->d;
  /* enumerate candidates in lexicographic order over [-r, r]^d, keep stars */
  int lim = 2 * radius + 1, total = 1;
  for (int i = 0; i < d; i++) total *= lim;
  for (int c = 0; c < total; c++) {
    int o[3] = {0, 0, 0}, rem = c, nz = 0;
    for (int i = d - 1; i >= 0; i--) {
      o[i] = rem % lim - radius;
      rem /= lim;
    }
    for (int i = 0; i < d; i++) nz += o[i] != 0;
    if (nz > 1) continue;
    f->term_array[t] = arr;
    for (int i = 0; i < 3; i++) f->term_off[t][i] = o[i];
    t++;
  }
  f->nterms = t;
}

static void add_term(sg_family* f, int arr, int o0, int o1, int o2) {
  int t = f->nterms++;
  f->term_array[t] = arr;
  f->term_off[t][0] = o0;
  f->term_off[t][1] = o1;
  f->term_off[t][2] = o2;
}

static void init_fams(void) {
  if (fams_ready) return;
  memset(FAMS, 0, sizeof(FAMS));
  sg_family* f;

  /* cfg 1: oracle/specs/wave1d.json */
  f = &FAMS[SG_WAVE1D];
  *f = (sg_family){.name = "wave1d", .d = 1, .lo = 1, .hi_n = -2, .shape_n = 0,
                   .nscalars = 1, .scalars = {"D"}, .narrays = 4,
                   .arrays = {"c", "u", "u_prev", "u_next"},
                   .adjoints = {"c_b", "u_b", "u_prev_b", "u_next_b"}, .output = 3,
                   .increment = 0, .radius = 1};
  add_term(f, 0, 0, 0, 0);
  add_term(f, 1, -1, 0, 0);
  add_term(f, 1, 0, 0, 0);
  add_term(f, 1, 1, 0, 0);
  add_term(f, 2, 0, 0, 0);

  /* cfg 2: oracle/specs/wave3d_c.json (bundled wave3d with c active) */
  for (int which = 0; which < 3; which++) {
    int id = which == 0 ? SG_WAVE3D_C : which == 1 ? SG_WAVE3D_C2 : SG_WAVE3D;
    f = &FAMS[id];
    *f = (sg_family){.name = which == 0 ? "wave3d_c" : which == 1 ? "wave3d_c2" : "wave3d",
                     .d = 3, .lo = 1, .hi_n = -2, .shape_n = 0, .nscalars = 1,
                     .scalars = {"D"}, .narrays = 4, .arrays = {"c", "u_1", "u_2", "u"},
                     .adjoints = {which == 2 ? "" : "c_b", "u_1_b", "u_2_b", "u_b"},
                     .output = 3, .increment = 1, .radius = 1};
    if (which != 2) add_term(f, 0, 0, 0, 0);
    set_terms_star(f, 1, 1, f->nterms);
    add_term(f, 2, 0, 0, 0);
  }

  /* cfg 3: oracle/specs/burgers2d.json */
  f = &FAMS[SG_BURGERS2D];
  *f = (sg_family){.name = "burgers2d", .d = 2, .lo = 1, .hi_n = -2, .shape_n = 0,
                   .nscalars = 2, .scalars = {"C", "D"}, .narrays = 2,
                   .arrays = {"u_1", "u"}, .adjoints = {"u_1_b", "u_b"}, .output = 1,
                   .increment = 0, .radius = 1};
  set_terms_star(f, 0, 1, 0);

  /* cfg 4/5: oracle/specs/wave3d_r4.json (u_2 passive) */
  f = &FAMS[SG_WAVE3D_R4];
  *f = (sg_family){.name = "wave3d_r4", .d = 3, .lo = 4, .hi_n = -5, .shape_n = 0,
                   .nscalars = 1, .scalars = {"D"}, .narrays = 4,
                   .arrays = {"c", "u_1", "u_2", "u"}, .adjoints = {"c_b", "u_1_b", "", "u_b"},
                   .output = 3, .increment = 0, .radius = 4};
  add_term(f, 0, 0, 0, 0);
  set_terms_star(f, 1, 4, 1);

  /* bundled lap1d (examples.cpp:9-26) */
  f = &FAMS[SG_LAP1D];
  *f = (sg_family){.name = "lap1d", .d = 1, .lo = 1, .hi_n = -1, .shape_n = 1, .nscalars = 0,
                   .narrays = 3, .arrays = {"c", "u", "r"}, .adjoints = {"", "ub", "rb"},
                   .output = 2, .increment = 0, .radius = 1};
  add_term(f, 1, -1, 0, 0);
  add_term(f, 1, 0, 0, 0);
  add_term(f, 1, 1, 0, 0);

  /* bundled burgers1d (examples.cpp:50-66) */
  f = &FAMS[SG_BURGERS1D];
  *f = (sg_family){.name = "burgers1d", .d = 1, .lo = 1, .hi_n = -2, .shape_n = 0,
                   .nscalars = 2, .scalars = {"C", "D"}, .narrays = 2, .arrays = {"u_1", "u"},
                   .adjoints = {"u_1_b", "u_b"}, .output = 1, .increment = 1, .radius = 1};
  add_term(f, 0, -1, 0, 0);
  add_term(f, 0, 0, 0, 0);
  add_term(f, 0, 1, 0, 0);
  fams_ready = 1;
}

const sg_family* sg_family_get(int fam) {
  init_fams();
  if (fam < 0 || fam >= SG_NUM_FAMILIES) return NULL;
  return &FAMS[fam];
}

int sg_family_by_name(const char* name) {
  init_fams();
  for (int i = 0; i < SG_NUM_FAMILIES; i++)
    if (strcmp(FAMS[i].name, name) == 0) return i;
  return -1;
}

long long sg_array_len(int fam, long long n) {
  const sg_family* f = sg_family_get(fam);
  long long e = n + f->shape_n, len = 1;
  for (int i = 0; i < f->d; i++) len *= e;
  return len;
}

/* ---------------- region splitting (adjoint.cpp:73-150) ---------------- */

typedef struct {
  int d, nterms;
  const int (*off)[3];
  const long long *lo, *hi;
  sg_nest* nests;
  int max_nests, count, core_index, overflow;
  long long plo[3], phi[3];
} split_ctx;

static void recurse(split_ctx* c, int dim, const int* alive, int nalive, int all_middle) {
  if (dim == c->d) {
    if (c->count >= c->max_nests) {
      c->overflow = 1;
      return;
    }
    sg_nest* n = &c->nests[c->count];
    for (int i = 0; i < c->d; i++) {
      n->lo[i] = c->plo[i];
      n->hi[i] = c->phi[i];
    }
    n->nterms = nalive;
    for (int i = 0; i < nalive; i++) n->terms[i] = alive[i];
    n->core = all_middle;
    if (all_middle) c->core_index = c->count;
    c->count++;
    return;
  }
  /* distinct offsets along dim, ascending (std::set, adjoint.cpp:92-94) */
  long long offs[SG_MAX_TERMS];
  int k = 0;
  for (int a = 0; a < nalive; a++) {
    long long o = c->off[alive[a]][dim];
    int seen = 0;
    for (int b = 0; b < k; b++) seen |= offs[b] == o;
    if (!seen) offs[k++] = o;
  }
  for (int a = 1; a < k; a++)
    for (int b = a; b > 0 && offs[b - 1] > offs[b]; b--) {
      long long t = offs[b];
      offs[b] = offs[b - 1];
      offs[b - 1] = t;
    }
  const long long s = c->lo[dim], e = c->hi[dim];
  int sub[SG_MAX_TERMS], ns;
  for (int j = 0; j + 1 < k; j++) { /* lower segments: terms with o <= offs[j] */
    c->plo[dim] = s + offs[j];
    c->phi[dim] = s + offs[j + 1] - 1;
    ns = 0;
    for (int a = 0; a < nalive; a++)
      if (c->off[alive[a]][dim] <= offs[j]) sub[ns++] = alive[a];
    recurse(c, dim + 1, sub, ns, 0);
  }
  c->plo[dim] = s + offs[k - 1]; /* middle */
  c->phi[dim] = e + offs[0];
  recurse(c, dim + 1, alive, nalive, all_middle);
  for (int j = 0; j + 1 < k; j++) { /* upper segments: terms with o > offs[j] */
    c->plo[dim] = e + offs[j] + 1;
    c->phi[dim] = e + offs[j + 1];
    ns = 0;
    for (int a = 0; a < nalive; a++)
      if (c->off[alive[a]][dim] > offs[j]) sub[ns++] = alive[a];
    recurse(c, dim + 1, sub, ns, 0);
  }
}

int sg_split_offsets(int d, int nterms, const int (*off)[3], const long long* lo,
                     const long long* hi, sg_nest* nests, int max_nests, int* core_index) {
  if (nterms <= 0 || nterms > SG_MAX_TERMS) return -1;
  split_ctx c = {.d = d, .nterms = nterms, .off = off, .lo = lo, .hi = hi, .nests = nests,
                 .max_nests = max_nests};
  int all[SG_MAX_TERMS];
  for (int i = 0; i < nterms; i++) all[i] = i;
  recurse(&c, 0, all, nterms, 1);
  if (c.overflow) return -1;
  if (core_index) *core_index = c.core_index;
  return c.count;
}

static void family_bounds(const sg_family* f, long long n, long long* lo, long long* hi) {
  for (int i = 0; i < f->d; i++) {
    lo[i] = f->lo;
    hi[i] = n + f->hi_n;
  }
}

int sg_split_family(int fam, long long n, sg_nest* nests, int max_nests, int* core_index) {
  const sg_family* f = sg_family_get(fam);
  long long lo[3], hi[3];
  family_bounds(f, n, lo, hi);
  return sg_split_offsets(f->d, f->nterms, (const int(*)[3])f->term_off, lo, hi, nests,
                          max_nests, core_index);
}

void sg_core_bounds(int fam, long long n, long long* lo, long long* hi) {
  const sg_family* f = sg_family_get(fam);
  long long plo[3], phi[3];
  family_bounds(f, n, plo, phi);
  for (int i = 0; i < f->d; i++) {
    int mx = f->term_off[0][i], mn = mx;
    for (int t = 0; t < f->nterms; t++) {
      if (f->term_off[t][i] > mx) mx = f->term_off[t][i];
      if (f->term_off[t][i] < mn) mn = f->term_off[t][i];
    }
    lo[i] = plo[i] + mx;
    hi[i] = phi[i] + mn;
  }
}

int sg_check_guards(int fam, long long n) {
  const sg_family* f = sg_family_get(fam);
  long long plo[3], phi[3];
  family_bounds(f, n, plo, phi);
  for (int i = 0; i < f->d; i++) {
    int mx = f->term_off[0][i], mn = mx;
    for (int t = 0; t < f->nterms; t++) {
      if (f->term_off[t][i] > mx) mx = f->term_off[t][i];
      if (f->term_off[t][i] < mn) mn = f->term_off[t][i];
    }
    if (mx - mn >= 1 && phi[i] - plo[i] < mx - mn) return 1;
  }
  return 0;
}

/* ---------------- partials and bodies (symdiff.cpp:238-305) ---------------- */

static inline long long flat(const sg_family* f, long long n, const long long* x) {
  long long e = n + f->shape_n, idx = 0;
  for (int i = 0; i < f->d; i++) idx = idx * e + x[i];
  return idx;
}

/* value of array a at x + (o0,o1,o2) */
static inline double at(const sg_family* f, const sg_env* env, int a, const long long* x, int o0,
                        int o1, int o2) {
  long long y[3] = {x[0] + o0, f->d > 1 ? x[1] + o1 : 0, f->d > 2 ? x[2] + o2 : 0};
  return env->grid[a][flat(f, env->n, y)];
}

static double lap7(const sg_family* f, const sg_env* env, int a, const long long* x) {
  return at(f, env, a, x, -1, 0, 0) + at(f, env, a, x, 0, -1, 0) + at(f, env, a, x, 0, 0, -1) -
         6.0 * at(f, env, a, x, 0, 0, 0) + at(f, env, a, x, 0, 0, 1) + at(f, env, a, x, 0, 1, 0) +
         at(f, env, a, x, 1, 0, 0);
}

static double lap25(const sg_family* f, const sg_env* env, int a, const long long* x) {
  double s = W4_CENTER3 * at(f, env, a, x, 0, 0, 0);
  for (int r = 1; r <= 4; r++)
    s += W4[r] * (at(f, env, a, x, -r, 0, 0) + at(f, env, a, x, r, 0, 0) +
                  at(f, env, a, x, 0, -r, 0) + at(f, env, a, x, 0, r, 0) +
                  at(f, env, a, x, 0, 0, -r) + at(f, env, a, x, 0, 0, r));
  return s;
}

static inline double sel_ge0(double v) { return v >= 0.0 ? 1.0 : 0.0; }

double sg_partial(int fam, const sg_env* env, int term, const long long* x) {
  const sg_family* f = sg_family_get(fam);
  const int* o = f->term_off[term];
  switch (fam) {
    case SG_WAVE1D: {
      const double D = env->scalars[0], c = at(f, env, 0, x, 0, 0, 0);
      if (term == 0) /* 2*D*(u[i-1] - 2.0*u[i] + u[i+1])*c[i] */
        return 2.0 * D *
               (at(f, env, 1, x, -1, 0, 0) - 2.0 * at(f, env, 1, x, 0, 0, 0) +
                at(f, env, 1, x, 1, 0, 0)) *
               c;
      if (term == 4) return -1.0;
      if (o[0] == 0) return -2.0 * D * c * c + 2.0;
      return D * c * c;
    }
    case SG_WAVE3D_C:
    case SG_WAVE3D_C2:
    case SG_WAVE3D: {
      const double D = env->scalars[0], c = at(f, env, 0, x, 0, 0, 0);
      const double cc = fam == SG_WAVE3D_C2 ? c * c : c;
      if (f->term_array[term] == 0) /* c_b term */
        return (fam == SG_WAVE3D_C2 ? 2.0 * D * c : D) * lap7(f, env, 1, x);
      if (f->term_array[term] == 2) return -1.0;
      if (o[0] == 0 && o[1] == 0 && o[2] == 0) return -6.0 * D * cc + 2.0;
      return D * cc;
    }
    case SG_WAVE3D_R4: {
      const double D = env->scalars[0], c = at(f, env, 0, x, 0, 0, 0);
      if (term == 0) return 2.0 * D * lap25(f, env, 1, x) * c;
      int r = abs(o[0]) + abs(o[1]) + abs(o[2]);
      if (r == 0) return W4_CENTER3 * D * c * c + 2.0;
      return W4[r] * D * c * c;
    }
    case SG_BURGERS2D: {
      const double C = env->scalars[0], D = env->scalars[1];
      const double u = at(f, env, 0, x, 0, 0, 0);
      if (o[0] < 0 || o[1] < 0) return C * fmax(0.0, u) + D;
      if (o[0] > 0 || o[1] > 0) return -C * fmin(0.0, u) + D;
      const double um = at(f, env, 0, x, -1, 0, 0), up = at(f, env, 0, x, 1, 0, 0);
      const double vm = at(f, env, 0, x, 0, -1, 0), vp = at(f, env, 0, x, 0, 1, 0);
      return -C * ((u - um) * sel_ge0(u) + (u - vm) * sel_ge0(u) + (vp - u) * sel_ge0(-u) +
                   (up - u) * sel_ge0(-u) + 2.0 * fmax(0.0, u) - 2.0 * fmin(0.0, u)) -
             4.0 * D + 1.0;
    }
    case SG_BURGERS1D: {
      const double C = env->scalars[0], D = env->scalars[1];
      const double u = at(f, env, 0, x, 0, 0, 0);
      if (o[0] < 0) return C * fmax(0.0, u) + D;
      if (o[0] > 0) return -C * fmin(0.0, u) + D;
      const double um = at(f, env, 0, x, -1, 0, 0), up = at(f, env, 0, x, 1, 0, 0);
      return -C * ((u - um) * sel_ge0(u) + (up - u) * sel_ge0(-u) + fmax(0.0, u) -
                   fmin(0.0, u)) -
             2.0 * D + 1.0;
    }
    case SG_LAP1D: {
      const double c = at(f, env, 0, x, 0, 0, 0);
      return (o[0] < 0 ? 2.0 : o[0] == 0 ? -3.0 : 4.0) * c;
    }
  }
  return 0.0;
}

double sg_body(int fam, const sg_env* env, const long long* x) {
  const sg_family* f = sg_family_get(fam);
  switch (fam) {
    case SG_WAVE1D: {
      const double D = env->scalars[0], c = at(f, env, 0, x, 0, 0, 0);
      const double u = at(f, env, 1, x, 0, 0, 0);
      return 2.0 * u - at(f, env, 2, x, 0, 0, 0) +
             c * c * D * (at(f, env, 1, x, -1, 0, 0) - 2.0 * u + at(f, env, 1, x, 1, 0, 0));
    }
    case SG_WAVE3D_C:
    case SG_WAVE3D_C2:
    case SG_WAVE3D: {
      const double D = env->scalars[0], c = at(f, env, 0, x, 0, 0, 0);
      const double cc = fam == SG_WAVE3D_C2 ? c * c : c;
      return 2.0 * at(f, env, 1, x, 0, 0, 0) - at(f, env, 2, x, 0, 0, 0) +
             cc * D * lap7(f, env, 1, x);
    }
    case SG_WAVE3D_R4: {
      const double D = env->scalars[0], c = at(f, env, 0, x, 0, 0, 0);
      return 2.0 * at(f, env, 1, x, 0, 0, 0) - at(f, env, 2, x, 0, 0, 0) +
             c * c * D * lap25(f, env, 1, x);
    }
    case SG_BURGERS2D: {
      const double C = env->scalars[0], D = env->scalars[1];
      const double u = at(f, env, 0, x, 0, 0, 0);
      const double um = at(f, env, 0, x, -1, 0, 0), up = at(f, env, 0, x, 1, 0, 0);
      const double vm = at(f, env, 0, x, 0, -1, 0), vp = at(f, env, 0, x, 0, 1, 0);
      return u -
             C * (fmax(u, 0.0) * (u - um) + fmin(u, 0.0) * (up - u) + fmax(u, 0.0) * (u - vm) +
                  fmin(u, 0.0) * (vp - u)) +
             D * (up + um + vp + vm - 4.0 * u);
    }
    case SG_BURGERS1D: {
      const double C = env->scalars[0], D = env->scalars[1];
      const double u = at(f, env, 0, x, 0, 0, 0);
      const double um = at(f, env, 0, x, -1, 0, 0), up = at(f, env, 0, x, 1, 0, 0);
      return u - C * (fmax(u, 0.0) * (u - um) + fmin(u, 0.0) * (up - u)) +
             D * (up + um - 2.0 * u);
    }
    case SG_LAP1D: {
      const double c = at(f, env, 0, x, 0, 0, 0);
      return c * (2.0 * at(f, env, 1, x, -1, 0, 0) - 3.0 * at(f, env, 1, x, 0, 0, 0) +
                  4.0 * at(f, env, 1, x, 1, 0, 0));
    }
  }
  return 0.0;
}

/* ---------------- executors (interp.cpp:131-228) ---------------- */

/* lexicographic iteration, outer slowest, inclusive bounds (interp.cpp:131-151) */
#define FOR_BOX(d, lo, hi, x)                                                        \
  for (x[0] = lo[0]; x[0] <= hi[0]; x[0]++)                                          \
    for (x[1] = (d > 1 ? lo[1] : 0); x[1] <= (d > 1 ? hi[1] : 0); x[1]++)            \
      for (x[2] = (d > 2 ? lo[2] : 0); x[2] <= (d > 2 ? hi[2] : 0); x[2]++)

static int seed_index(const sg_family* f) { return f->output; }

int sg_run_primal(int fam, sg_env* env) {
  const sg_family* f = sg_family_get(fam);
  long long lo[3], hi[3], x[3];
  family_bounds(f, env->n, lo, hi);
  double* out = env->grid[f->output];
  FOR_BOX(f->d, lo, hi, x) {
    double v = sg_body(fam, env, x);
    long long k = flat(f, env->n, x);
    if (f->increment)
      out[k] += v;
    else
      out[k] = v;
  }
  return 0;
}

static inline void gather_term(const sg_family* f, int fam, sg_env* env, int t,
                               const long long* y) {
  long long xs[3] = {y[0] - f->term_off[t][0], f->d > 1 ? y[1] - f->term_off[t][1] : 0,
                     f->d > 2 ? y[2] - f->term_off[t][2] : 0};
  const double* seed = env->adj[seed_index(f)];
  double v = sg_partial(fam, env, t, xs) * seed[flat(f, env->n, xs)];
  env->adj[f->term_array[t]][flat(f, env->n, y)] += v;
}

int sg_run_program(int fam, sg_env* env) {
  const sg_family* f = sg_family_get(fam);
  if (sg_check_guards(fam, env->n)) return 1;
  static sg_nest nests[SG_MAX_NESTS];
  int core;
  int nn = sg_split_family(fam, env->n, nests, SG_MAX_NESTS, &core);
  if (nn < 0) return -1;
  for (int k = 0; k < nn; k++) {
    const sg_nest* ns = &nests[k];
    long long x[3];
    FOR_BOX(f->d, ns->lo, ns->hi, x) {
      for (int a = 0; a < ns->nterms; a++) gather_term(f, fam, env, ns->terms[a], x);
    }
  }
  return 0;
}

static inline int in_box(const sg_family* f, const long long* lo, const long long* hi,
                         const long long* y, int t) {
  for (int i = 0; i < f->d; i++) {
    long long v = y[i] - f->term_off[t][i];
    if (v < lo[i] || v > hi[i]) return 0;
  }
  return 1;
}

int sg_run_program_predicate(int fam, sg_env* env) {
  const sg_family* f = sg_family_get(fam);
  if (sg_check_guards(fam, env->n)) return 1;
  long long lo[3], hi[3], wlo[3] = {0, 0, 0}, whi[3] = {0, 0, 0}, y[3];
  family_bounds(f, env->n, lo, hi);
  for (int i = 0; i < f->d; i++) whi[i] = env->n + f->shape_n - 1;
  FOR_BOX(f->d, wlo, whi, y) {
    for (int t = 0; t < f->nterms; t++)
      if (in_box(f, lo, hi, y, t)) gather_term(f, fam, env, t, y);
  }
  return 0;
}

int sg_run_program_omp(int fam, sg_env* env) {
  const sg_family* f = sg_family_get(fam);
  if (sg_check_guards(fam, env->n)) return -1;
  long long lo[3], hi[3], whi[3] = {0, 0, 0};
  family_bounds(f, env->n, lo, hi);
  for (int i = 0; i < f->d; i++) whi[i] = env->n + f->shape_n - 1;
  int threads = 1;
#pragma omp parallel
  {
#ifdef _OPENMP
#pragma omp single
    threads = omp_get_num_threads();
#endif
#pragma omp for schedule(static)
    for (long long i0 = 0; i0 <= whi[0]; i0++) {
      long long y[3];
      y[0] = i0;
      for (y[1] = 0; y[1] <= whi[1]; y[1]++)
        for (y[2] = 0; y[2] <= whi[2]; y[2]++)
          for (int t = 0; t < f->nterms; t++)
            if (in_box(f, lo, hi, y, t)) gather_term(f, fam, env, t, y);
    }
  }
  return threads;
}

int sg_run_scatter(int fam, sg_env* env) {
  const sg_family* f = sg_family_get(fam);
  long long lo[3], hi[3], x[3];
  family_bounds(f, env->n, lo, hi);
  const double* seed = env->adj[seed_index(f)];
  FOR_BOX(f->d, lo, hi, x) {
    double sd = seed[flat(f, env->n, x)];
    for (int t = 0; t < f->nterms; t++) {
      double s = sg_partial(fam, env, t, x);
      long long y[3] = {x[0] + f->term_off[t][0], x[1] + f->term_off[t][1],
                        x[2] + f->term_off[t][2]};
      env->adj[f->term_array[t]][flat(f, env->n, y)] += s * sd;
    }
  }
  return 0;
}

double sg_max_rel_err(const double* a, const double* b, long long len) {
  double worst = 0.0;
  for (long long i = 0; i < len; i++) {
    double e = fabs(a[i] - b[i]) / (1.0 + fabs(b[i]));
    if (e > worst || e != e) worst = e;
  }
  return worst;
}
