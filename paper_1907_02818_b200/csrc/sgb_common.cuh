// Shared helpers for the sm_100a adjoint-stencil kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "stencilgrad_b200.h"

namespace sgb {

// 8th-order second-derivative weights, identical literals to
// oracle/specs/wave3d_r4.json; W4C3 is 3*w0 as the reference folds it.
__host__ __device__ constexpr double w4(int r) {
  return r == 0 ? -2.8472222222222223
                : r == 1 ? 1.6 : r == 2 ? -0.2 : r == 3 ? 0.025396825396825397 : -0.0017857142857142857;
}
constexpr double kW4C3 = -8.541666666666668;

// Stencil families (match oracle family ids where they overlap).
enum Family : int { WAVE1D = 0, WAVE3D_C = 1, WAVE3D_C2 = 2, BURGERS2D = 3, WAVE3D_R4 = 4 };

// Per-thread error text + global launch counter (host side).
void set_error(const std::string& msg);
extern std::atomic<unsigned long long> g_launches;

inline int launch_status(const char* what) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return -static_cast<int>(e);
  }
  return 0;
}

inline cudaStream_t as_stream(sgb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

// Radius-R star on a cube: write box of the gather adjoint for target arrays
// reached by every star offset is the primal box dilated along one axis at a
// time (a point is reached iff at most one coordinate is outside [lo, hi] and
// that one by at most R).  See SURVEY Appendix C.
__device__ __forceinline__ bool in_range(long long v, long long lo, long long hi) {
  return v >= lo && v <= hi;
}

template <int R>
__device__ __forceinline__ bool star_reached(long long i, long long j, long long k, long long lo,
                                             long long hi) {
  const int oi = (i < lo) ? (int)(lo - i) : (i > hi) ? (int)(i - hi) : 0;
  const int oj = (j < lo) ? (int)(lo - j) : (j > hi) ? (int)(j - hi) : 0;
  const int ok = (k < lo) ? (int)(lo - k) : (k > hi) ? (int)(k - hi) : 0;
  const int nout = (oi > 0) + (oj > 0) + (ok > 0);
  return nout == 0 || (nout == 1 && oi <= R && oj <= R && ok <= R);
}

// ---- launcher state (runtime.cu) --------------------------------------------
// Run-time options: scheduling / A-B knobs whose defaults are the measured
// best.  Read from the environment (SGB_<NAME>) once per process, changed
// afterwards only through sgb_set_option; no launcher calls getenv.
#define SGB_OPTIONS(X)                                                                     \
  X(STAR_KERNEL)      /* 1 | 7: force the radius-1 or radius-4 streaming design */       \
  X(F64_PLANE)        /* fp64 radius 4 on the plane kernels */                          \
  X(GENERIC_POINT)    /* per-point 3D gather kernels */                                 \
  X(PLANE_NO_TMA)     /* plane kernel without TMA */                                    \
  X(PRIMAL_GENERIC)   /* per-point primal kernels */                                    \
  X(BURGERS_NORING)   /* burgers2d register-streaming kernels */                        \
  X(BURGERS_RING_RB)  /* rows per CTA of the burgers2d ring gather */                   \
  X(BURGERS_RING_S)   /* ring stages of the burgers2d gather */                         \
  X(BURGERS_RB)       /* rows per CTA of the burgers2d streaming gather */              \
  X(BURGERS_PRIMAL_RB)                                                                   \
  X(BURGERS_PRIMAL_S)                                                                    \
  X(FRESH_UNFUSED)    /* fresh entries as memset + accumulating gather */               \
  X(STEP_UNFUSED)     /* time-loop step as gather + box set */                          \
  X(PLAN_CHUNKS)      /* i-chunks of the host-buffer pipeline */                        \
  X(F64_ICHUNKS)      /* i-chunks of the fp64 streaming gather */                       \
  X(PRIMAL_CHUNKS)    /* i-chunks of the 3D primals */                                  \
  X(PLANE_CHUNK)      /* planes per CTA of the plane kernels */                         \
  X(NO_UBWIN)         /* in-kernel seed mask instead of the windowed TMA map */         \
  X(ICHUNKS)          /* i-chunks of the radius-4 interior (or unified) launch */       \
  X(ICHUNKS_F)        /* i-chunks of the radius-4 frame launch */                       \
  X(V7_UNIFIED)       /* radius 4: one launch for frame + interior */                   \
  X(V7_SPLIT)         /* radius 4: two launches even for partial plane ranges */        \
  X(FORK)             /* radius 4: frame launch on a side stream */                     \
  X(DISABLE_TMA)      /* no TMA kernels */                                              \
  X(L2PROMO)          /* TMA L2 promotion bytes (0, 64, 128, 256) */                    \
  X(V7_PREFETCH)      /* radius 4: L2 prefetch distance beyond the smem ring, planes */ \
  X(V8_INTERIOR)      /* radius 4: the 4-row-per-thread interior kernel (0 | 1) */     \
  X(F64_V8)           /* fp64 radius 4: the 4-row-per-thread streaming kernel (0 | 1) */ \
  X(V8_FRAME)         /* radius 4, v8 on: the frame tiles in v8 as well */              \
  X(V8_BALANCE)       /* radius 4, v8 interior: balanced last wave (0 off, 1 on) */      \
  X(R1_FP64ACC)       /* radius-1 fp32 gathers accumulate in fp64 (default 1) */

#define SGB_OPT_ENUM(n) OPT_##n,
enum Opt : int { SGB_OPTIONS(SGB_OPT_ENUM) kNumOpts };
#undef SGB_OPT_ENUM
#define SGB_OPT_NAME(n) #n,
static constexpr const char* kOptNames[] = {SGB_OPTIONS(SGB_OPT_NAME)};
#undef SGB_OPT_NAME

long long opt(Opt o, long long dflt);  // the set value, else dflt
bool opt_flag(Opt o);                  // set and non-zero
int num_sms();                         // SMs of the current device (cached per device)
// dynamic shared-memory attribute of `fn` on the current device, set once per
// (device, kernel); 0 or a negative error (sgb_last_error set)
int ensure_smem(const void* fn, size_t bytes, const char* what);
// a CUDA driver entry point by name (cudaGetDriverEntryPoint, cached; nullptr
// if unavailable) -- the library keeps no link-time libcuda dependency for it
void* driver_entry(const char* name);

inline unsigned grid_1d(long long work, int block) {
  long long g = (work + block - 1) / block;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace sgb
