/* stencilgrad_b200.h — C ABI of the B200 (sm_100a) adjoint-stencil library.
 *
 * Drop-in for the functions the reference's C/OpenMP emitter generates
 * (/root/reference/proj/src/codegen.cpp): same names, same parameter order
 * (every size symbol, then each referenced scalar as double, then each
 * referenced array in declaration order with each primal followed by its
 * adjoint; codegen.cpp:198-230), with three B200 differences:
 *   - a dtype suffix (_f32 / _f64): arrays are float* or double*;
 *   - array pointers are DEVICE pointers (cudaMalloc / torch CUDA memory);
 *   - a trailing stream (cudaStream_t passed as void*; NULL = legacy stream).
 * Calls are stream-ordered and asynchronous; the caller synchronises.
 *
 * Semantics (codegen.cpp:332-434, interp.cpp:183-228):
 *   <name>           primal: out (=|+=) body over the primal box
 *                    (emit_primal, codegen.cpp:311-330; run_nest, interp.hpp:56)
 *   <name>_b         gather adjoint: every adjoint array is ACCUMULATED (+=),
 *                    core + boundary regions of assemble_adjoint
 *                    (adjoint.cpp:152-163) fused into one launch; points that
 *                    no term reaches are left untouched
 *                    (emit_adjoint, codegen.cpp:332-382; run_program, interp.hpp:59)
 *   <name>_scatter_b scatter adjoint with atomics (ablation only)
 *                    (emit_scatter_adjoint, codegen.cpp:384-434;
 *                    run_scatter_adjoint, interp.hpp:63)
 * Return codes: 0 success; 1 minimum-extent guard violated (checked on the
 * host before any launch, as the emitted `if ( n - 3 < 2 ) return 1;`,
 * codegen.cpp:353-357); negative: -(cudaError_t) of a failed launch, or
 * SGB_EINVAL for an argument outside the supported domain (never a CPU
 * fallback).  sgb_last_error() describes the last failure on this thread.
 */
#ifndef STENCILGRAD_B200_H
#define STENCILGRAD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* sgb_stream_t; /* cudaStream_t */

#define SGB_OK 0
#define SGB_GUARD 1
#define SGB_EINVAL (-10000)

const char* sgb_last_error(void);
const char* sgb_version(void);
/* number of kernel launches issued by this library since load (all threads) */
unsigned long long sgb_launch_count(void);

/* ---- run-time options ---------------------------------------------------------
 * Scheduling / A-B knobs (kernel variant, i-chunking, ...) whose defaults are
 * the measured best; none selects a CPU path.  The environment (SGB_<NAME>)
 * is read once, at the first call that needs an option; afterwards options
 * change only through these calls (thread-safe, process-wide).  Names are
 * listed by sgb_option_name(0 .. ) (NULL past the end); an "SGB_" prefix is
 * accepted.  Unknown names return SGB_EINVAL. */
int sgb_set_option(const char* name, long long value);
int sgb_clear_option(const char* name);
int sgb_get_option(const char* name, long long* value, int* is_set);
const char* sgb_option_name(int index);

/* ---- program-keyed dispatch ---------------------------------------------------
 * The hand-tuned kernels of a family compute ONE AdjointProgram: the
 * reference front end's assemble_adjoint (adjoint.cpp:152-163, adjoint.hpp:37-45)
 * of oracle/specs/<family>.json.  sgb_program_family(text) returns the family
 * whose kernels compute exactly the program whose canonical text is given, or
 * NULL (sgb_last_error names the closest family and the first differing
 * line) -- callers holding an AdjointProgram dispatch through this instead of
 * a name, and lower any other program with the NVRTC emitter.  Canonical text
 * (one item per line, as printed by b200_program_text in
 * oracle/ref/b200_binding.cpp):
 *   sgb-program 1
 *   counters <c0> <c1> ...
 *   guard <hi - lo (AffineExpr::str)> >= <needed>          per dimension
 *   term <t> read <array> offset <o..> adjoint <a_b> seed <seed>[<c>].. partial <to_input_string>
 *   valid <t> <lo>:<hi>,...                                 per shifted statement
 *   nest <lo>:<hi>,... terms <t..>[ core]                   per nest, program order
 *   core <core_index>
 * sgb_program_text(family): the embedded text; sgb_family_signature(family):
 * "<sizes>;<scalars>;<arrays>" of the generated <family>_b prototype
 * (codegen.cpp:198-230), comma-separated, e.g. "n;D;c,c_b,u_1,u_1_b,u_b".
 * None of these needs a GPU. */
const char* sgb_program_family(const char* canonical_text);
const char* sgb_program_text(const char* family);
const char* sgb_family_signature(const char* family);

/* ---- cfg 1: wave1d (oracle/specs/wave1d.json) -------------------------------
 * u_next[i] = 2u[i] - u_prev[i] + c[i]^2 D (u[i-1] - 2u[i] + u[i+1]), i in [1, n-2]
 * Reference prototypes: wave1d(int n, double D, double *c, double *u,
 * double *u_prev, double *u_next); wave1d_b(int n, double D, double *c,
 * double *c_b, double *u, double *u_b, double *u_prev_b, double *u_next_b). */
int wave1d_f64(int n, double D, double* c, double* u, double* u_prev, double* u_next,
               sgb_stream_t stream);
int wave1d_b_f64(int n, double D, double* c, double* c_b, double* u, double* u_b,
                 double* u_prev_b, double* u_next_b, sgb_stream_t stream);
int wave1d_scatter_b_f64(int n, double D, double* c, double* c_b, double* u, double* u_b,
                         double* u_prev_b, double* u_next_b, sgb_stream_t stream);
int wave1d_f32(int n, double D, float* c, float* u, float* u_prev, float* u_next,
               sgb_stream_t stream);
int wave1d_b_f32(int n, double D, float* c, float* c_b, float* u, float* u_b, float* u_prev_b,
                 float* u_next_b, sgb_stream_t stream);
int wave1d_scatter_b_f32(int n, double D, float* c, float* c_b, float* u, float* u_b,
                         float* u_prev_b, float* u_next_b, sgb_stream_t stream);
/* wave1d_b restricted to the outputs j in [j0, j1) (n, j0, j1 even, 16-byte
 * aligned arrays): inputs [j0-1, j1] must be resident.  The chunk unit of the
 * pipelined host-buffer plan. */
int wave1d_b_range_f64(int n, double D, double* c, double* c_b, double* u, double* u_b,
                       double* u_prev_b, double* u_next_b, long long j0, long long j1,
                       sgb_stream_t stream);
int wave1d_b_range_f32(int n, double D, float* c, float* c_b, float* u, float* u_b,
                       float* u_prev_b, float* u_next_b, long long j0, long long j1,
                       sgb_stream_t stream);

/* ---- cfg 2: wave3d_c, 7-point star, linear c (oracle/specs/wave3d_c.json) ---
 * u[i][j][k] += 2u_1 - u_2 + c D Lap7(u_1), box [1, n-2]^3.
 * Reference prototype: wave3d_c_b(int n, double D, double *c, double *c_b,
 * double *u_1, double *u_1_b, double *u_2_b, double *u_b).
 * wave3d_c2 is the c^2 variant (oracle/specs/wave3d_c2.json), same ABI. */
int wave3d_c_f32(int n, double D, float* c, float* u_1, float* u_2, float* u,
                 sgb_stream_t stream);
int wave3d_c_b_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                   float* u_2_b, float* u_b, sgb_stream_t stream);
int wave3d_c_scatter_b_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                           float* u_2_b, float* u_b, sgb_stream_t stream);
int wave3d_c_f64(int n, double D, double* c, double* u_1, double* u_2, double* u,
                 sgb_stream_t stream);
int wave3d_c_b_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                   double* u_2_b, double* u_b, sgb_stream_t stream);
int wave3d_c_scatter_b_f64(int n, double D, double* c, double* c_b, double* u_1,
                           double* u_1_b, double* u_2_b, double* u_b, sgb_stream_t stream);
int wave3d_c2_f32(int n, double D, float* c, float* u_1, float* u_2, float* u,
                  sgb_stream_t stream);
int wave3d_c2_b_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                    float* u_2_b, float* u_b, sgb_stream_t stream);
int wave3d_c2_scatter_b_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                            float* u_2_b, float* u_b, sgb_stream_t stream);
int wave3d_c2_f64(int n, double D, double* c, double* u_1, double* u_2, double* u,
                  sgb_stream_t stream);
int wave3d_c2_b_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                    double* u_2_b, double* u_b, sgb_stream_t stream);
int wave3d_c2_scatter_b_f64(int n, double D, double* c, double* c_b, double* u_1,
                            double* u_1_b, double* u_2_b, double* u_b, sgb_stream_t stream);

/* ---- cfg 3: burgers2d (oracle/specs/burgers2d.json) --------------------------
 * Reference prototype: burgers2d_b(int n, double C, double D, double *u_1,
 * double *u_1_b, double *u_b). */
int burgers2d_f64(int n, double C, double D, double* u_1, double* u, sgb_stream_t stream);
int burgers2d_b_f64(int n, double C, double D, double* u_1, double* u_1_b, double* u_b,
                    sgb_stream_t stream);
int burgers2d_scatter_b_f64(int n, double C, double D, double* u_1, double* u_1_b,
                            double* u_b, sgb_stream_t stream);
int burgers2d_f32(int n, double C, double D, float* u_1, float* u, sgb_stream_t stream);
int burgers2d_b_f32(int n, double C, double D, float* u_1, float* u_1_b, float* u_b,
                    sgb_stream_t stream);
int burgers2d_scatter_b_f32(int n, double C, double D, float* u_1, float* u_1_b, float* u_b,
                            sgb_stream_t stream);
/* burgers2d_b restricted to output rows [row0, row1) (rows a 16-byte
 * multiple, aligned arrays): rows row0-1 .. row1 must be resident. */
int burgers2d_b_rows_f64(int n, double C, double D, double* u_1, double* u_1_b, double* u_b,
                         int row0, int row1, sgb_stream_t stream);
int burgers2d_b_rows_f32(int n, double C, double D, float* u_1, float* u_1_b, float* u_b,
                         int row0, int row1, sgb_stream_t stream);

/* ---- cfg 4/5: wave3d_r4, 8th-order 25-point star (oracle/specs/wave3d_r4.json)
 * u = 2u_1 - u_2 + c^2 D Lap25(u_1), box [4, n-5]^3; u_2 passive.
 * Reference prototypes: wave3d_r4(int n, double D, double *c, double *u_1,
 * double *u_2, double *u); wave3d_r4_b(int n, double D, double *c,
 * double *c_b, double *u_1, double *u_1_b, double *u_b). */
int wave3d_r4_f32(int n, double D, float* c, float* u_1, float* u_2, float* u,
                  sgb_stream_t stream);
int wave3d_r4_b_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                    float* u_b, sgb_stream_t stream);
int wave3d_r4_scatter_b_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                            float* u_b, sgb_stream_t stream);
int wave3d_r4_f64(int n, double D, double* c, double* u_1, double* u_2, double* u,
                  sgb_stream_t stream);
int wave3d_r4_b_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                    double* u_b, sgb_stream_t stream);
int wave3d_r4_scatter_b_f64(int n, double D, double* c, double* c_b, double* u_1,
                            double* u_1_b, double* u_b, sgb_stream_t stream);

/* ---- z-slab (outermost counter i) entry points for multi-GPU decomposition --
 * Local arrays hold planes [i_base, i_base + nplanes) of the global n^3 grid
 * (n*n contiguous elements per plane).  Computes the gather adjoint for the
 * global output planes [out_i0, out_i1), which must lie within
 * [i_base + R, i_base + nplanes - R) unless they touch the global grid ends
 * (R = stencil radius).  Bounds masks use GLOBAL indices, so the union of
 * the slabs' outputs equals the single-GPU result bit for bit. */
int wave3d_r4_b_slab_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                         float* u_b, int i_base, int nplanes, int out_i0, int out_i1,
                         sgb_stream_t stream);
/* Fused halo exchange: the same z-slab adjoint, but the local arrays hold
 * exactly the planes [i_base, i_base + nplanes) and every input plane below /
 * above them is read straight from the lower / upper neighbour's arrays
 * (lo_* / hi_*, holding global planes [lo_base, lo_base + lo_nplanes) /
 * [hi_base, ...); NULL at a grid end) by the kernel's own TMA loads -- peer
 * memory over NVLink when the pointers come from sgb_ipc_open, no separate
 * send/recv.  The neighbours' planes must be final before the call. */
int wave3d_r4_b_slab_peer_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                              float* u_b, int i_base, int nplanes, int out_i0, int out_i1,
                              const float* lo_c, const float* lo_u_1, const float* lo_u_b,
                              int lo_base, int lo_nplanes, const float* hi_c,
                              const float* hi_u_1, const float* hi_u_b, int hi_base,
                              int hi_nplanes, sgb_stream_t stream);
/* CUDA IPC for the fused path: a 64-byte handle (+ byte offset) of the device
 * allocation holding ptr; open maps a peer's allocation into this process */
int sgb_ipc_handle(const void* ptr, void* handle64, long long* offset);
int sgb_ipc_open(const void* handle64, long long offset, void** ptr);
int sgb_ipc_close(void* ptr, long long offset);
int wave3d_c_b_slab_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                        float* u_2_b, float* u_b, int i_base, int nplanes, int out_i0,
                        int out_i1, sgb_stream_t stream);
/* fp64 forms of the z-slab entries (the reference's precision; host-buffer
 * plan chunks, multi-GPU slabs) */
int wave3d_r4_b_slab_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                         double* u_b, int i_base, int nplanes, int out_i0, int out_i1,
                         sgb_stream_t stream);
int wave3d_c_b_slab_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                        double* u_2_b, double* u_b, int i_base, int nplanes, int out_i0,
                        int out_i1, sgb_stream_t stream);

/* ---- multi-GPU z-slab plan ---------------------------------------
 * One rank per GPU owns the global planes [own0, own1) of the outermost
 * counter (sgb_slab_decompose: balanced contiguous split, R halo planes on
 * interior sides; local arrays hold planes [base, base + nplanes)).  The plan
 * owns the communication and a comm stream; the caller owns and binds every
 * array of <family>_b (set 0; the inputs c / u_1 / u_b may get a second
 * buffer set 1 for pipelining -- unbound set-1 arrays fall back to set 0).
 * Transports (no reference counterpart: the reference is single-node CPU,
 * SPEC.md:8):
 *   SGB_TRANSPORT_NCCL  ncclSend / ncclRecv of the R edge planes to rank +- 1
 *                       in one group on the comm stream; every rank passes the
 *                       same 128-byte ncclUniqueId (sgb_nccl_unique_id on one
 *                       rank, broadcast out of band); libnccl.so.2 dlopen'ed.
 *   SGB_TRANSPORT_IPC   each rank maps its neighbours' arrays (CUDA IPC, peer
 *                       memory over NVLink) and pushes its edge planes into
 *                       their halos with copy engines; ordering by stream
 *                       memory operations on epoch flags, no host round trip.
 *                       Blobs are exchanged out of band: every rank calls
 *                       sgb_slab_ipc_export after binding, then connects with
 *                       its lower / upper neighbour's blob (NULL at grid ends).
 * sgb_slab_halo_start(set, mask): refresh the halo planes of the fields in
 * mask (1 = c, 2 = u_1, 4 = u_b) of `set`, ordered after the work queued on
 * `stream`, asynchronously on the comm stream; every prior reader of those
 * halos must be ordered before it on `stream`.  sgb_slab_halo_wait makes
 * `stream` wait for it (incoming halos arrived, outgoing planes sent).
 * sgb_slab_step: one reverse step over the owned planes -- exchange u_1 / u_b,
 * then the gather (flags: SGB_STEP_OVERLAP = interior planes during the
 * exchange, then the two edge bands; SGB_STEP_FRESH = u_1_b written as the
 * step's adjoint alone (wave3d_r4 fp32); SGB_STEP_NO_EXCHANGE = the halos of
 * `set` were refreshed by an earlier sgb_slab_halo_start (pipelined drivers):
 * wait for it, then one launch).  All calls are collective in order: every
 * rank issues the same sequence. */
#define SGB_TRANSPORT_NCCL 1
#define SGB_TRANSPORT_IPC 2
#define SGB_STEP_FRESH 1
#define SGB_STEP_OVERLAP 2
#define SGB_STEP_NO_EXCHANGE 4
typedef struct sgb_slab sgb_slab;
int sgb_slab_decompose(int n, int radius, int world, int rank, int* own0, int* own1, int* base,
                       int* nplanes);
int sgb_nccl_unique_id(void* id128);
sgb_slab* sgb_slab_create(const char* family, int n, int dtype_bytes, int rank, int world,
                          int transport, const void* nccl_id128);
int sgb_slab_geometry(const sgb_slab* plan, int* base, int* nplanes, int* own0, int* own1);
int sgb_slab_bind(sgb_slab* plan, int set, const char* name, void* device_ptr);
/* blob == NULL: *bytes = the blob size */
int sgb_slab_ipc_export(const sgb_slab* plan, void* blob, long long* bytes);
int sgb_slab_ipc_connect(sgb_slab* plan, const void* lower_blob, const void* upper_blob);
/* Connection probe (collective, after every rank connected): phase 0 writes
 * this rank's token into each neighbour's probe words, once by a stream memory
 * operation and once by a copy-engine copy (the two paths the exchange uses;
 * neither can block); phase 1, after all ranks finished phase 0 (out-of-band
 * barrier), checks that both neighbours' tokens arrived -- an error means the
 * box has no usable peer path and the IPC transport must not be used. */
int sgb_slab_ipc_probe(sgb_slab* plan, int phase);
/* Watchdog's last resort for an IPC plan whose exchange never completed:
 * satisfies every wait on this rank's epoch flags from a fresh stream so the
 * queued work drains; the plan's results are void and it must be destroyed. */
int sgb_slab_release(sgb_slab* plan);
int sgb_slab_halo_start(sgb_slab* plan, int set, unsigned fields_mask, sgb_stream_t stream);
int sgb_slab_halo_wait(sgb_slab* plan, int set, sgb_stream_t stream);
int sgb_slab_step(sgb_slab* plan, int set, const double* scalars, int flags,
                  sgb_stream_t stream);
void sgb_slab_destroy(sgb_slab* plan);

/* ---- device input generation (synthetic BASELINE distributions) -------------
 * Counter-based: value(index) depends only on (seed, stream, global index), so
 * any slab of any decomposition sees identical inputs.  index = global flat
 * index of dst[0] is index_base.  kind: 0 = N(mean, scale), 1 = U[mean, mean+scale)
 * (i.e. lo = mean, width = scale). */
int sgb_fill_random_f32(float* dst, long long count, long long index_base, uint64_t seed,
                        uint64_t stream_id, int kind, double mean, double scale,
                        sgb_stream_t stream);
int sgb_fill_random_f64(double* dst, long long count, long long index_base, uint64_t seed,
                        uint64_t stream_id, int kind, double mean, double scale,
                        sgb_stream_t stream);
/* N(mean, scale^2) on planes [i_base, i_base+nplanes) of an n^3 grid with the
 * h-point shell set to zero (one fused pass; same counter-based values as
 * sgb_fill_random_f32 at the same global indices) */
int sgb_fill_normal3d_f32(float* dst, int n, int i_base, int nplanes, int halo, uint64_t seed,
                          uint64_t stream_id, double mean, double scale, sgb_stream_t stream);
/* the same values widened to fp64 (the fp64 forms of the 3D configurations
 * see exactly the fp32 inputs) */
int sgb_fill_normal3d_f64(double* dst, int n, int i_base, int nplanes, int halo, uint64_t seed,
                          uint64_t stream_id, double mean, double scale, sgb_stream_t stream);
/* two fields in one pass (cfg 5 regenerates u_1 and the seed every step):
 * bitwise the values of sgb_fill_normal3d_* (a, halo_a, stream_a) and
 * (b, halo_b, stream_b) over the same planes */
int sgb_fill_normal3d_pair_f32(float* a, int halo_a, uint64_t stream_a, float* b, int halo_b,
                               uint64_t stream_b, int n, int i_base, int nplanes, uint64_t seed,
                               double mean, double scale, sgb_stream_t stream);
int sgb_fill_normal3d_pair_f64(double* a, int halo_a, uint64_t stream_a, double* b, int halo_b,
                               uint64_t stream_b, int n, int i_base, int nplanes, uint64_t seed,
                               double mean, double scale, sgb_stream_t stream);
/* zero the h-point shell of planes [i_base, i_base+nplanes) of an n^d grid
 * (d = 1, 2 or 3; for d < 3 pass i_base = 0, nplanes = n) */
int sgb_zero_halo_f32(float* a, int d, int n, int h, int i_base, int nplanes,
                      sgb_stream_t stream);
int sgb_zero_halo_f64(double* a, int d, int n, int h, int i_base, int nplanes,
                      sgb_stream_t stream);
/* c[i][j][k] = value of layer floor(i*layers/n), layer values ~ U[lo, hi) from seed */
int sgb_fill_layered_f32(float* c, int n, int layers, double lo, double hi, uint64_t seed,
                         int i_base, int nplanes, sgb_stream_t stream);
/* y += alpha x on the box [lo, hi]^3 of local planes [i_base, i_base+nplanes):
 * the u_2 term of a full time-loop adjoint (u-bar^{t-1} -= u-bar^{t+1} on B) */
int sgb_box_axpy_f32(float* y, const float* x, double alpha, int n, int lo, int hi, int i_base,
                     int nplanes, sgb_stream_t stream);
int sgb_box_axpy_f64(double* y, const double* x, double alpha, int n, int lo, int hi,
                     int i_base, int nplanes, sgb_stream_t stream);
/* y = alpha x on the box, 0 elsewhere (a zeroed y followed by box_axpy, in one
 * pass) on local planes [i_base, i_base+nplanes) */
int sgb_box_set_f32(float* y, const float* x, double alpha, int n, int lo, int hi, int i_base,
                    int nplanes, sgb_stream_t stream);
int sgb_box_set_f64(double* y, const double* x, double alpha, int n, int lo, int hi, int i_base,
                    int nplanes, sgb_stream_t stream);
/* One reverse step of a wave3d_r4 time loop (drivers.time_loop_adjoint; no
 * reference counterpart -- the reference's scope ends at one loop nest,
 * SPEC.md:8): the gather adjoint wave3d_r4_b (c_b, u_1_b accumulated) and
 * the u_2 partial u_2_b = -u_b on [4, n-5]^3, 0 elsewhere, in one pass
 * (bitwise = wave3d_r4_b_f32 followed by sgb_box_set_f32(u_2_b, u_b, -1)). */
int sgb_wave3d_r4_b_step_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                             float* u_b, float* u_2_b, sgb_stream_t stream);
/* wave3d_r4_b with u_1_b = this call's adjoint alone (c_b accumulated as
 * usual): the fused form of zeroing u_1_b and calling wave3d_r4_b_f32 --
 * bitwise equal -- for independent reverse steps (BASELINE cfg 5; no
 * reference counterpart).  The slab form works on local planes like
 * wave3d_r4_b_slab_f32 and writes the output planes [out_i0, out_i1). */
int wave3d_r4_b_fresh_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                              float* u_b, sgb_stream_t stream);
int wave3d_r4_b_fresh_slab_f32(int n, double D, float* c, float* c_b, float* u_1,
                                   float* u_1_b, float* u_b, int i_base, int nplanes,
                                   int out_i0, int out_i1, sgb_stream_t stream);
/* the same at the reference's precision (fp64 streaming kernel, MODE 4) */
int wave3d_r4_b_fresh_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                          double* u_b, sgb_stream_t stream);
int wave3d_r4_b_fresh_slab_f64(int n, double D, double* c, double* c_b, double* u_1,
                               double* u_1_b, double* u_b, int i_base, int nplanes, int out_i0,
                               int out_i1, sgb_stream_t stream);
/* wave3d_c_b / wave3d_c2_b with u_2_b = this call's u_2 partial alone (-u_b
 * on [1, n-2]^3, 0 elsewhere; c_b, u_1_b accumulated): the zeroing of u_2_b
 * a carried reverse sweep does after rotating its adjoints, fused -- bitwise
 * equal to zeroing u_2_b and calling the accumulating entry. */
int wave3d_c_b_fresh_u2_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                            float* u_2_b, float* u_b, sgb_stream_t stream);
int wave3d_c2_b_fresh_u2_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                             float* u_2_b, float* u_b, sgb_stream_t stream);
/* one interior pass of the 5-point average u <- (u + 4 neighbours)/5 (2D) */
int sgb_smooth5_f64(const double* src, double* dst, int n, sgb_stream_t stream);

/* ---- device-side parity reductions (verification entries; synchronous) -----
 * compare_grids of the reference (interp.cpp:290-298) on DEVICE arrays, a in
 * the kernel's precision, b the fp64 oracle grid uploaded to the device:
 * out4[0] = max_i |a_i - b_i| / (1 + |b_i|) over finite terms, out4[1] =
 * sum (a - b)^2, out4[2] = sum b^2 (the norm metric), out4[3] = number of
 * non-finite terms (a pass needs 0).  fp64 accumulation, deterministic.
 * sgb_dot_*: <a, b> in fp64, the inner products of dot_product_test
 * (interp.cpp:354-375). */
int sgb_compare_f32(const float* a, const double* b, long long count, double* out4,
                    sgb_stream_t stream);
int sgb_compare_f64(const double* a, const double* b, long long count, double* out4,
                    sgb_stream_t stream);
int sgb_dot_f32(const float* a, const float* b, long long count, double* out,
                sgb_stream_t stream);
int sgb_dot_f64(const double* a, const double* b, long long count, double* out,
                sgb_stream_t stream);

/* ---- host-buffer entry (end-to-end path) ------------------------------------
 * Same arguments as <name>_b but HOST pointers; copies inputs and accumulated
 * adjoints host->device, runs the gather adjoint, copies the adjoints back.
 * A plan owns the device workspace so the call itself does not allocate. */
typedef struct sgb_plan sgb_plan;
sgb_plan* sgb_plan_create(const char* family, int n, int dtype_bytes);
/* z-slab plan (multi-GPU host-buffer path): the host arrays hold local planes
 * [i_base, i_base + nplanes) of the global n^3 grid; the call computes the
 * gather adjoint of global output planes [out_i0, out_i1) (wave3d_r4 /
 * wave3d_c, fp32), H2D / kernel / D2H pipelined over i-chunks */
sgb_plan* sgb_plan_create_slab(const char* family, int n, int dtype_bytes, int i_base,
                               int nplanes, int out_i0, int out_i1);
void sgb_plan_destroy(sgb_plan* plan);
/* arrays[] in the reference prototype order of <family>_b (host pointers) */
int sgb_plan_run_adjoint_host(sgb_plan* plan, const double* scalars, void** arrays,
                              sgb_stream_t stream);
/* Reverse sweeps over HOST-held forward states (the multi-step BASELINE
 * protocols with the states checkpointed in host memory rather than
 * regenerated).  The reference's CPU sweep calls <name>_b (codegen.cpp:332-382)
 * once per step with everything staying in host RAM; here whatever does not
 * change per step stays RESIDENT on the device between begin and end.
 * arrays[] are host pointers in the prototype order of <family>_b; every call
 * returns with its copies complete.
 *   wave3d_r4 plans (cfg 5, independent steps; fp32 / fp64, grid or slab;
 *   c, c_b, u_1, u_1_b, u_b): begin reads c, c_b; a step reads u_1, u_b and
 *   writes u_1_b = the step's own adjoint (12 instead of 28 bytes per point
 *   over PCIe in fp32); end writes the accumulated c_b.  Bitwise = zeroing
 *   u_1_b and calling sgb_plan_run_adjoint_host per step.
 *   wave3d_c full-grid plans (cfg 2, carried steps; c, c_b, u_1, u_1_b, u_2_b,
 *   u_b): begin reads c, c_b, u_1_b, u_2_b and the seed u_b; a step reads only
 *   the state u_1 (4 instead of 36 bytes per point), accumulates c_b, u_1_b,
 *   u_2_b and rotates the adjoints on the device (seed <- u_1_b, u_1_b <-
 *   u_2_b, u_2_b <- 0); end writes c_b, u_1_b, u_2_b and the current seed u_b.
 *   Bitwise = the per-step accumulating call followed by the caller's rotation.
 * While a sweep is open sgb_plan_run_adjoint_host on the same plan is refused
 * (it would overwrite the resident arrays). */
int sgb_plan_sweep_begin(sgb_plan* plan, void** arrays, sgb_stream_t stream);
int sgb_plan_sweep_step_host(sgb_plan* plan, const double* scalars, void** arrays,
                             sgb_stream_t stream);
int sgb_plan_sweep_end(sgb_plan* plan, void** arrays, sgb_stream_t stream);

/* ---- emitted kernels (runtime compilation) ----------------
 * paper_1907_02818_b200/emitter.py generates CUDA source for the fused gather
 * adjoint / primal of ANY problem the reference front end differentiates (its
 * AdjointProgram: terms, offsets, partials); these entry points compile it
 * with NVRTC for sm_100a (cached by source text) and launch it. */
typedef struct sgb_jit_kernel sgb_jit_kernel;
const char* sgb_jit_log(void);
int sgb_jit_compile(const char* source, const char* name, sgb_jit_kernel** out);
/* compile-only check (no GPU needed): 0 when the source compiles for sm_100a */
int sgb_jit_check(const char* source);
int sgb_jit_launch(sgb_jit_kernel* kernel, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                   unsigned by, unsigned bz, void** args, sgb_stream_t stream);
/* the same with `smem` bytes of dynamic shared memory */
int sgb_jit_launch_smem(sgb_jit_kernel* kernel, unsigned gx, unsigned gy, unsigned gz,
                        unsigned bx, unsigned by, unsigned bz, unsigned smem, void** args,
                        sgb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
