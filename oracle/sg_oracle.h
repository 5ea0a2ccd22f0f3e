/* sg_oracle.h — CPU restatement of the reference's adjoint-stencil semantics.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker (or the timed CPU port).  The product path
 * (paper_1907_02818_b200) never links or calls it.
 *
 * Parity is pinned: tests/test_oracle_pins.py checks this restatement against
 * (1) the reference's own known-answer tests (nest counts 5/53/25/125/17,
 * test_adjoint.cpp:137-151; lap1d five regions :112-135; core bounds
 * :96-110; guards :225-233) and (2) golden vectors produced by the unmodified
 * reference library (oracle/_ref/ref_harness, run_program / run_scatter_adjoint
 * / run_nest) committed under tests/golden/.
 *
 * All grids are dense row-major fp64 with the innermost counter contiguous
 * (interp.cpp:30-35, codegen.cpp:40-57).
 */
#ifndef SG_ORACLE_H
#define SG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_MAX_TERMS 32
#define SG_MAX_NESTS 4096
#define SG_MAX_ARRAYS 6

/* Families: the BASELINE config encodings (oracle/specs/<family>.json) plus the
 * reference's bundled examples (examples.cpp:9-66) used for pinning. */
enum {
  SG_WAVE1D = 0,    /* cfg 1 */
  SG_WAVE3D_C = 1,  /* cfg 2 (linear c, bundled wave3d with c active) */
  SG_WAVE3D_C2 = 2, /* cfg 2 alternative (c^2) */
  SG_BURGERS2D = 3, /* cfg 3 */
  SG_WAVE3D_R4 = 4, /* cfg 4, 5 */
  SG_LAP1D = 5,     /* bundled example lap1d */
  SG_WAVE3D = 6,    /* bundled example wave3d (c passive) */
  SG_BURGERS1D = 7, /* bundled example burgers1d */
  SG_NUM_FAMILIES = 8
};

/* Static description of one family, mirroring Problem + derive_adjoint_terms
 * (nest.hpp:55-61, adjoint.cpp:9-25). */
typedef struct {
  const char* name;
  int d;                          /* nest depth (counters outer -> inner) */
  int lo;                         /* primal bounds [lo, n + hi_n] per dim  */
  int hi_n;                       /*   (all families use the same per dim) */
  int shape_n;                    /* array extent = n + shape_n per dim    */
  int nscalars;
  const char* scalars[2];
  int narrays;                    /* declaration order is significant      */
  const char* arrays[SG_MAX_ARRAYS];
  const char* adjoints[SG_MAX_ARRAYS]; /* "" when passive                  */
  int output;                     /* index of the lhs (output) array       */
  int increment;                  /* primal mode: 1 for +=, 0 for =        */
  int nterms;                     /* active_reads order (symdiff.cpp:204)  */
  int term_array[SG_MAX_TERMS];   /* read array index                      */
  int term_off[SG_MAX_TERMS][3];  /* offset vector, outer first            */
  int radius;                     /* max |offset| over all terms           */
} sg_family;

const sg_family* sg_family_get(int fam);
int sg_family_by_name(const char* name);

/* Environment: primal grids and adjoint grids indexed like family->arrays. */
typedef struct {
  long long n;
  double scalars[2];
  double* grid[SG_MAX_ARRAYS];
  double* adj[SG_MAX_ARRAYS];
} sg_env;

/* One hierarchical nest (adjoint.cpp:73-120). */
typedef struct {
  long long lo[3], hi[3];
  int nterms;
  int terms[SG_MAX_TERMS];
  int core;
} sg_nest;

/* Restatement of split_regions/Splitter::recurse (adjoint.cpp:73-150) on an
 * explicit offset list (nterms offsets of depth d, bounds [lo, hi] per dim).
 * Writes up to max_nests nests; returns the number of nests, or -1 on overflow.
 * *core_index receives the index of the all-middle nest. */
int sg_split_offsets(int d, int nterms, const int (*off)[3], const long long* lo,
                     const long long* hi, sg_nest* nests, int max_nests, int* core_index);

/* Family-level helpers. */
int sg_split_family(int fam, long long n, sg_nest* nests, int max_nests, int* core_index);
void sg_core_bounds(int fam, long long n, long long* lo, long long* hi);   /* adjoint.cpp:55-69 */
/* Extent guards (adjoint.cpp:134-143): returns 0 when all hold, 1 otherwise. */
int sg_check_guards(int fam, long long n);
long long sg_array_len(int fam, long long n);

/* S_l evaluated at primal point x (the partials of symdiff.cpp:296-305). */
double sg_partial(int fam, const sg_env* env, int term, const long long* x);
/* The primal rhs at x. */
double sg_body(int fam, const sg_env* env, const long long* x);

/* run_nest (interp.cpp:153-187): primal, in place on env->grid[output]. */
int sg_run_primal(int fam, sg_env* env);
/* run_program (interp.cpp:189-198): guards, then the hierarchical nests in
 * program order, lexicographic points, statements in ascending term order. */
int sg_run_program(int fam, sg_env* env);
/* Predicate form of the same program: for every y of the
 * write box, for l ascending, if y - o_l in B: adj_l[y] += S_l(y-o_l) seed[y-o_l].
 * Bitwise identical to sg_run_program because each cell sees the same ordered
 * sequence of increments. */
int sg_run_program_predicate(int fam, sg_env* env);
/* run_scatter_adjoint (interp.cpp:200-228). */
int sg_run_scatter(int fam, sg_env* env);
/* OpenMP-parallel predicate-form gather (the "port" CPU baseline); returns the
 * number of threads used. */
int sg_run_program_omp(int fam, sg_env* env);

/* compare_grids (interp.cpp:290-298): max |a-b| / (1+|b|). */
double sg_max_rel_err(const double* a, const double* b, long long len);

#ifdef __cplusplus
}
#endif
#endif
