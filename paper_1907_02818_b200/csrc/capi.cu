// extern "C" entry points (include/stencilgrad_b200.h): argument checks, the
// reference's minimum-extent guards, and dispatch to the sm_100a kernels.
#include <cstdio>
#include <type_traits>
#include <cstring>
#include <string>
#include <vector>

#include "generic_kernels.cuh"
#include "lowdim.cuh"
#include "star3d_plane.cuh"
#include "star3d_primal.cuh"
#include "star3d_r4.cuh"
#include "star3d_f64.cuh"
#include "star3d_tma.cuh"

namespace sgb {

std::atomic<unsigned long long> g_launches{0};
static thread_local std::string t_error;
void set_error(const std::string& msg) { t_error = msg; }

template <typename A, typename B, typename C, typename E>
static bool aligned16(const A* a, const B* b, const C* c, const E* e) {
  return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) |
           reinterpret_cast<uintptr_t>(c) | reinterpret_cast<uintptr_t>(e)) & 15) == 0;
}
template <typename A, typename B>
static bool aligned16(const A* a, const B* b) {
  return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
}

static int einval(const std::string& msg) {
  set_error(msg);
  return SGB_EINVAL;
}

// Minimum-extent guard of split_regions (adjoint.cpp:134-143), as the emitted
// code checks it (codegen.cpp:353-357): (hi - lo) >= max o - min o per dim.
static bool guard_ok(int fam, long long n) {
  switch (fam) {
    case WAVE1D:
    case WAVE3D_C:
    case WAVE3D_C2:
    case BURGERS2D:
      return (n - 3) >= 2;  // [1, n-2], offsets -1..1
    case WAVE3D_R4:
      return (n - 9) >= 8;  // [4, n-5], offsets -4..4
  }
  return false;
}

// ------------------------------------------------------------------ 3D stars
// Kernel selection for the TMA path ("Measured path"): the
// radius-4 streaming kernel (v7) for radius 4, the v1 streaming kernel for
// radius 1 (measured faster there); SGB_STAR_KERNEL=1|7 forces one of them.
static int star_kernel_version(int mode) {
  const long long v = opt(OPT_STAR_KERNEL, 0);
  if (v == 1 || v == 7) return (int)v;
  return mode == 2 ? 7 : 1;
}

template <int MODE, typename T>
static int star3_gather(const char* name, long long n, double D, const T* c, T* c_b,
                        const T* u_1, T* u_1_b, T* u_2_b, const T* u_b, long long i_base,
                        long long nplanes, long long out_i0, long long out_i1,
                        cudaStream_t s) {
  using S = Star3<MODE>;
  constexpr int R = S::R;
  const int fam = MODE == 0 ? WAVE3D_C : MODE == 1 ? WAVE3D_C2 : WAVE3D_R4;
  if (n <= 0) return einval(std::string(name) + ": n must be positive");
  if (!guard_ok(fam, n)) return SGB_GUARD;
  if (!c || !c_b || !u_1 || !u_1_b || !u_b || (S::kU2 && !u_2_b))
    return einval(std::string(name) + ": null array");
  if (out_i0 < 0 || out_i1 > n || out_i0 > out_i1 || nplanes <= 0)
    return einval(std::string(name) + ": bad output plane range");
  const long long need_lo = out_i0 - R < 0 ? 0 : out_i0 - R;
  const long long need_hi = out_i1 - 1 + R > n - 1 ? n - 1 : out_i1 - 1 + R;
  if (out_i1 > out_i0 && (need_lo < i_base || need_hi >= i_base + nplanes))
    return einval(std::string(name) + ": slab does not hold the radius-R halo of the outputs");
  if (out_i1 == out_i0) return 0;
  const long long lo = R, hi = n - 1 - R;
  Slab3 g{n, i_base, nplanes};
  if (star3_tma_ok<MODE, T>(n, {c, c_b, u_1, u_1_b, u_2_b, u_b})) {
    if (star_kernel_version(MODE) == 7)
      return star3_v7_gather<MODE>(g, lo, hi, out_i0, out_i1, (float)D, (const float*)c,
                                   (float*)c_b, (const float*)u_1, (float*)u_1_b, (float*)u_2_b,
                                   (const float*)u_b, s, name);
    if constexpr (MODE < 2) {
      if (opt(OPT_R1_FP64ACC, 1))  // radius-1 specs: fp64 accumulation
        return star3_tma_gather<MODE, false, true>(g, lo, hi, out_i0, out_i1, D,
                                                   (const float*)c, (float*)c_b,
                                                   (const float*)u_1, (float*)u_1_b,
                                                   (float*)u_2_b, (const float*)u_b, s, name);
    }
    return star3_tma_gather<MODE>(g, lo, hi, out_i0, out_i1, D, (const float*)c,
                                  (float*)c_b, (const float*)u_1, (float*)u_1_b,
                                  (float*)u_2_b, (const float*)u_b, s, name);
  }
  // plane-streaming kernel for radius 4 (measured: fp64 768^3 29 -> ~12 ms);
  // radius 1 keeps the per-point kernel (measured faster there)
  if constexpr (std::is_same<T, double>::value) {
    // fp64: the register-blocked streaming kernel (star3d_f64.cuh)
    if (!opt_flag(OPT_F64_PLANE) && !opt_flag(OPT_GENERIC_POINT) && n <= 46340) {
      const int rc = star3_f64_stream_gather<MODE>(g, lo, hi, out_i0, out_i1, D, c, c_b, u_1,
                                                   u_1_b, u_2_b, u_b, s, name);
      if (rc != 1) return rc;
    }
  }
  if (MODE == 2 && !opt_flag(OPT_GENERIC_POINT) && n <= 46340) {
    if (!opt_flag(OPT_PLANE_NO_TMA)) {
      const int rc = star3_plane_tma_gather<MODE, T>(g, lo, hi, out_i0, out_i1, (T)D, c, c_b,
                                                     u_1, u_1_b, u_2_b, u_b, s, name);
      if (rc != 1) return rc;
    }
    return star3_plane_gather<MODE, T>(g, lo, hi, out_i0, out_i1, (T)D, c, c_b, u_1, u_1_b,
                                       u_2_b, u_b, s, name);
  }
  dim3 b(32, 4), gr((unsigned)((n + 31) / 32), (unsigned)((n + 3) / 4),
                    (unsigned)(out_i1 - out_i0));
  star3_gather_kernel<MODE, T>
      <<<gr, b, 0, s>>>(g, lo, hi, out_i0, out_i1, (T)D, c, c_b, u_1, u_1_b, u_2_b, u_b);
  return launch_status(name);
}

template <int MODE, typename T>
static int star3_primal(const char* name, long long n, double D, const T* c, const T* u_1,
                        const T* u_2, T* u, cudaStream_t s) {
  constexpr int R = Star3<MODE>::R;
  if (n <= 0) return einval(std::string(name) + ": n must be positive");
  if (!c || !u_1 || !u_2 || !u) return einval(std::string(name) + ": null array");
  if (n < 2 * R + 1) return 0;  // empty primal box
  if (std::is_same<T, float>::value && !opt_flag(OPT_PRIMAL_GENERIC)) {
    const int rc = star3_primal_tma<MODE>(n, (float)D, (const float*)c, (const float*)u_1,
                                          (const float*)u_2, (float*)u, s, name);
    if (rc != 1) return rc;  // 1: TMA path not applicable (alignment / size)
  }
  if constexpr (std::is_same<T, double>::value && MODE == 2) {
    // radius 4 (the radius-1 fp64 primal is already at the copy bandwidth on
    // the per-point kernel)
    if (!opt_flag(OPT_PRIMAL_GENERIC)) {
      const int rc = star3_primal_f64_stream<MODE>(n, D, c, u_1, u_2, u, s, name);
      if (rc != 1) return rc;
    }
  }
  const long long lo = R, hi = n - 1 - R;
  dim3 b(32, 4), gr((unsigned)((n + 31) / 32), (unsigned)((n + 3) / 4), (unsigned)n);
  star3_primal_kernel<MODE, T><<<gr, b, 0, s>>>(Slab3{n, 0, n}, lo, hi, 0, n, (T)D, c, u_1,
                                                u_2, u);
  return launch_status(name);
}

template <int MODE, typename T>
static int star3_scatter(const char* name, long long n, double D, const T* c, T* c_b,
                         const T* u_1, T* u_1_b, T* u_2_b, const T* u_b, cudaStream_t s) {
  using S = Star3<MODE>;
  constexpr int R = S::R;
  if (n <= 0) return einval(std::string(name) + ": n must be positive");
  if (!c || !c_b || !u_1 || !u_1_b || !u_b || (S::kU2 && !u_2_b))
    return einval(std::string(name) + ": null array");
  const long long lo = R, hi = n - 1 - R;
  if (hi < lo) return 0;
  const long long m = hi - lo + 1;
  dim3 b(32, 4), gr((unsigned)((m + 31) / 32), (unsigned)((m + 3) / 4), (unsigned)m);
  star3_scatter_kernel<MODE, T>
      <<<gr, b, 0, s>>>(Slab3{n, 0, n}, lo, hi, (T)D, c, c_b, u_1, u_1_b, u_2_b, u_b);
  return launch_status(name);
}

// ------------------------------------------------------------------ wave1d
// Output range [j0, j1) of the streaming kernel (the range entries and the
// pipelined host plan); needs n, j0, j1 even and 16-byte aligned arrays.
template <typename T>
static bool wave1d_range_ok(long long n, long long j0, long long j1, const void* c,
                            const void* c_b, const void* u, const void* u_b, const void* u_prev_b,
                            const void* u_next_b) {
  return n % 2 == 0 && j0 % 2 == 0 && j1 % 2 == 0 && 0 <= j0 && j0 <= j1 && j1 <= n &&
         aligned16(c, c_b, u, u_b) && aligned16(u_prev_b, u_next_b);
}

template <typename T>
static int wave1d_gather(long long n, double D, const T* c, T* c_b, const T* u, T* u_b,
                         T* u_prev_b, const T* u_next_b, cudaStream_t s, long long j0 = 0,
                         long long j1 = -1) {
  if (n <= 0) return einval("wave1d_b: n must be positive");
  if (!guard_ok(WAVE1D, n)) return SGB_GUARD;
  if (!c || !c_b || !u || !u_b || !u_prev_b || !u_next_b) return einval("wave1d_b: null array");
  const bool range = j1 >= 0;
  if (!range) j1 = n;
  if (wave1d_range_ok<T>(n, j0, j1, c, c_b, u, u_b, u_prev_b, u_next_b)) {
    if (j1 == j0) return 0;
    wave1d_stream_kernel<T><<<grid_1d((j1 - j0) / 2, 256), 256, 0, s>>>(
        n, (T)D, c, c_b, u, u_b, u_prev_b, u_next_b, j0, j1);
    return launch_status("wave1d_b");
  }
  if (range) return einval("wave1d_b_range: needs even n, j0, j1 and 16-byte aligned arrays");
  wave1d_gather_kernel<T>
      <<<grid_1d(n, 256), 256, 0, s>>>(n, (T)D, c, c_b, u, u_b, u_prev_b, u_next_b);
  return launch_status("wave1d_b");
}

// ------------------------------------------------------------------ burgers2d
template <typename T>
static int burgers2d_gather(long long n, double C, double D, const T* u_1, T* u_1_b,
                            const T* u_b, cudaStream_t s, int row_lo = 0, int row_hi = -1) {
  if (n <= 0) return einval("burgers2d_b: n must be positive");
  if (!guard_ok(BURGERS2D, n)) return SGB_GUARD;
  if (!u_1 || !u_1_b || !u_b) return einval("burgers2d_b: null array");
  const bool range = row_hi >= 0;
  if (!range) row_hi = (int)n;
  if (range && (row_lo < 0 || row_lo > row_hi || row_hi > n))
    return einval("burgers2d_b_rows: bad row range");
  if ((n * (long long)sizeof(T)) % 16 == 0 && n <= (1 << 30) && aligned16(u_1, u_1_b, u_b, u_b) &&
      (range || !opt_flag(OPT_BURGERS_NORING))) {
    if (row_hi == row_lo) return 0;
    // rows per CTA / ring stages: measured defaults (options override)
    const int rb = (int)std::max<long long>(1, opt(OPT_BURGERS_RING_RB, 32));
    const int stages = (int)opt(OPT_BURGERS_RING_S, 5);
    int rc = 0;
    if (stages == 4)
      rc = ensure_smem((const void*)burgers2d_ring_kernel<T, 4>, BurgRing<T, 4>::SMEM, "burgers2d_b");
    else if (stages == 5)
      rc = ensure_smem((const void*)burgers2d_ring_kernel<T, 5>, BurgRing<T, 5>::SMEM, "burgers2d_b");
    else if (stages == 6)
      rc = ensure_smem((const void*)burgers2d_ring_kernel<T, 6>, BurgRing<T, 6>::SMEM, "burgers2d_b");
    else
      rc = ensure_smem((const void*)burgers2d_ring_kernel<T, 8>, BurgRing<T, 8>::SMEM, "burgers2d_b");
    if (rc) return rc;
    constexpr int W = BurgRing<T>::W, TH = BurgRing<T>::THREADS;
    dim3 g((unsigned)((n + W - 1) / W), (unsigned)((row_hi - row_lo + rb - 1) / rb));
    if (stages == 4)
      burgers2d_ring_kernel<T, 4><<<g, TH, BurgRing<T, 4>::SMEM, s>>>(
          (int)n, (T)C, (T)D, u_1, u_1_b, u_b, rb, row_lo, row_hi);
    else if (stages == 5)
      burgers2d_ring_kernel<T, 5><<<g, TH, BurgRing<T, 5>::SMEM, s>>>(
          (int)n, (T)C, (T)D, u_1, u_1_b, u_b, rb, row_lo, row_hi);
    else if (stages == 6)
      burgers2d_ring_kernel<T, 6><<<g, TH, BurgRing<T, 6>::SMEM, s>>>(
          (int)n, (T)C, (T)D, u_1, u_1_b, u_b, rb, row_lo, row_hi);
    else
      burgers2d_ring_kernel<T, 8><<<g, TH, BurgRing<T, 8>::SMEM, s>>>(
          (int)n, (T)C, (T)D, u_1, u_1_b, u_b, rb, row_lo, row_hi);
    return launch_status("burgers2d_b");
  }
  if (range) return einval("burgers2d_b_rows: needs 16-byte rows and aligned arrays");
  if (n % 2 == 0 && aligned16(u_1, u_1_b, u_b, u_b)) {
    long long rb = opt(OPT_BURGERS_RB, 32);  // rows per block, measured default
    if (rb <= 0) rb = 32;
    dim3 g((unsigned)((n / 2 + 127) / 128), (unsigned)((n + rb - 1) / rb));
    burgers2d_stream_kernel<T><<<g, 128, 0, s>>>(n, (T)C, (T)D, u_1, u_1_b, u_b, rb);
    return launch_status("burgers2d_b");
  }
  dim3 b(64, 4), g((unsigned)((n + 63) / 64), (unsigned)((n + 3) / 4));
  burgers2d_gather_kernel<T><<<g, b, 0, s>>>(n, (T)C, (T)D, u_1, u_1_b, u_b);
  return launch_status("burgers2d_b");
}

// burgers2d primal, strip-streaming ring kernel (lowdim.cuh).  Returns true
// when it launched (the caller checks the launch status), false when the
// shape needs the register-streaming / per-point kernels.
template <typename T>
static bool burgers2d_primal_ring(long long n, double C, double D, const T* u_1, T* u,
                                  cudaStream_t s) {
  if ((n * (long long)sizeof(T)) % 16 != 0 || n > (1 << 30) || !aligned16(u_1, u, u_1, u) ||
      opt_flag(OPT_BURGERS_NORING))
    return false;
  // measured at 8192^2; options override
  const int rb = (int)std::max<long long>(1, opt(OPT_BURGERS_PRIMAL_RB, 16));
  const long long sv = opt(OPT_BURGERS_PRIMAL_S, 6);
  const int stages = sv <= 4 ? 4 : (sv >= 8 ? 8 : 6);
  const int rc = stages == 4 ? ensure_smem((const void*)burgers2d_primal_ring_kernel<T, 4>,
                                           BurgPrimalRing<T, 4>::SMEM, "burgers2d")
                 : stages == 6 ? ensure_smem((const void*)burgers2d_primal_ring_kernel<T, 6>,
                                             BurgPrimalRing<T, 6>::SMEM, "burgers2d")
                               : ensure_smem((const void*)burgers2d_primal_ring_kernel<T, 8>,
                                             BurgPrimalRing<T, 8>::SMEM, "burgers2d");
  if (rc) return false;
  constexpr int W = BurgPrimalRing<T, 4>::W, TH = BurgPrimalRing<T, 4>::THREADS;
  dim3 g((unsigned)((n + W - 1) / W), (unsigned)((n + rb - 1) / rb));
  if (stages == 4)
    burgers2d_primal_ring_kernel<T, 4>
        <<<g, TH, BurgPrimalRing<T, 4>::SMEM, s>>>((int)n, (T)C, (T)D, u_1, u, rb);
  else if (stages == 6)
    burgers2d_primal_ring_kernel<T, 6>
        <<<g, TH, BurgPrimalRing<T, 6>::SMEM, s>>>((int)n, (T)C, (T)D, u_1, u, rb);
  else
    burgers2d_primal_ring_kernel<T, 8>
        <<<g, TH, BurgPrimalRing<T, 8>::SMEM, s>>>((int)n, (T)C, (T)D, u_1, u, rb);
  return true;
}

// wave3d_c / wave3d_c2 gather whose u_2_b is this call's u_2 partial alone
// (0 - u_b on the box, 0 elsewhere): the carried reverse sweep's zeroing of
// u_2_b after its rotation, fused (v1 streaming kernel, U2SET).
template <int MODE>
static int star3_c_fresh_u2(const char* name, int n, double D, float* c, float* c_b,
                            float* u_1, float* u_1_b, float* u_2_b, float* u_b,
                            cudaStream_t s) {
  if (n <= 0) return einval(std::string(name) + ": n must be positive");
  if (!guard_ok(MODE == 0 ? WAVE3D_C : WAVE3D_C2, n)) return SGB_GUARD;
  if (!c || !c_b || !u_1 || !u_1_b || !u_2_b || !u_b)
    return einval(std::string(name) + ": null array");
  // the fused U2SET form exists in the v1 kernel only: a forced radius-4
  // design (SGB_STAR_KERNEL=7) takes the zero-then-accumulate form below, so
  // this entry stays bitwise equal to adjoint() under every kernel choice
  if (star3_tma_ok<MODE, float>(n, {c, c_b, u_1, u_1_b, u_2_b, u_b}) &&
      !opt_flag(OPT_FRESH_UNFUSED) && star_kernel_version(MODE) != 7)
  {
    if (opt(OPT_R1_FP64ACC, 1))
      return star3_tma_gather<MODE, true, true>(Slab3{n, 0, n}, 1, n - 2, 0, n, D, c, c_b,
                                                u_1, u_1_b, u_2_b, u_b, s, name);
    return star3_tma_gather<MODE, true>(Slab3{n, 0, n}, 1, n - 2, 0, n, D, c, c_b, u_1,
                                        u_1_b, u_2_b, u_b, s, name);
  }
  // other shapes: zero u_2_b, then the accumulating gather
  if (cudaMemsetAsync(u_2_b, 0, (size_t)n * n * n * sizeof(float), s) != cudaSuccess)
    return launch_status(name);
  return star3_gather<MODE, float>(name, n, D, c, c_b, u_1, u_1_b, u_2_b, u_b, 0, n, 0, n, s);
}

// wave3d_r4 gather with u_1_b = this call's adjoint alone (MODE 4 of the
// radius-4 streaming kernels, fp32 and fp64), on local planes [i_base,
// i_base + nplanes), outputs [out_i0, out_i1).
template <typename T>
static int r4_fresh(const char* name, int n, double D, T* c, T* c_b, T* u_1, T* u_1_b, T* u_b,
                    long long i_base, long long nplanes, long long out_i0, long long out_i1,
                    cudaStream_t s) {
  constexpr int R = 4;
  if (n <= 0 || nplanes <= 0) return einval(std::string(name) + ": bad sizes");
  if (!guard_ok(WAVE3D_R4, n)) return SGB_GUARD;
  if (!c || !c_b || !u_1 || !u_1_b || !u_b) return einval(std::string(name) + ": null array");
  if (out_i0 < 0 || out_i1 > n || out_i0 > out_i1 || i_base < 0 || i_base + nplanes > n ||
      out_i0 < i_base || out_i1 > i_base + nplanes)
    return einval(std::string(name) + ": bad output plane range");
  const long long need_lo = out_i0 - R < 0 ? 0 : out_i0 - R;
  const long long need_hi = out_i1 - 1 + R > n - 1 ? n - 1 : out_i1 - 1 + R;
  if (out_i1 > out_i0 && (need_lo < i_base || need_hi >= i_base + nplanes))
    return einval(std::string(name) + ": slab does not hold the radius-R halo of the outputs");
  if (out_i1 == out_i0) return 0;
  if (!opt_flag(OPT_FRESH_UNFUSED)) {
    if constexpr (std::is_same<T, float>::value) {
      if (star3_tma_ok<4, float>(n, {c, c_b, u_1, u_1_b, u_b}))
        return star3_v7_gather<4>(Slab3{n, i_base, nplanes}, R, n - 1 - R, out_i0, out_i1,
                                  (float)D, c, c_b, u_1, u_1_b, nullptr, u_b, s, name);
    } else {
      if (!opt_flag(OPT_F64_PLANE) && !opt_flag(OPT_GENERIC_POINT)) {
        const int rc = star3_f64_stream_gather<4>(Slab3{n, i_base, nplanes}, R, n - 1 - R,
                                                  out_i0, out_i1, D, c, c_b, u_1, u_1_b,
                                                  nullptr, u_b, s, name);
        if (rc != 1) return rc;  // 1: shape / alignment not taken by the kernel
      }
    }
  }
  // other shapes: zero the output planes of u_1_b, then the accumulating gather
  const size_t plane = (size_t)n * n;
  if (cudaMemsetAsync(u_1_b + (out_i0 - i_base) * plane, 0,
                      (size_t)(out_i1 - out_i0) * plane * sizeof(T), s) != cudaSuccess)
    return launch_status(name);
  return star3_gather<2, T>(name, n, D, c, c_b, u_1, u_1_b, nullptr, u_b, i_base, nplanes,
                            out_i0, out_i1, s);
}

}  // namespace sgb

using namespace sgb;

extern "C" {

const char* sgb_last_error(void) { return t_error.c_str(); }
const char* sgb_version(void) { return "stencilgrad_b200 0.1 sm_100a"; }
unsigned long long sgb_launch_count(void) { return g_launches.load(); }

// ---- wave1d
#define SGB_WAVE1D(T, SFX)                                                                     \
  int wave1d_##SFX(int n, double D, T* c, T* u, T* u_prev, T* u_next, sgb_stream_t stream) {   \
    if (n <= 0 || !c || !u || !u_prev || !u_next) return einval("wave1d: bad arguments");      \
    wave1d_primal_kernel<T><<<grid_1d(n, 256), 256, 0, as_stream(stream)>>>(n, (T)D, c, u,     \
                                                                             u_prev, u_next);  \
    return launch_status("wave1d");                                                            \
  }                                                                                            \
  int wave1d_b_##SFX(int n, double D, T* c, T* c_b, T* u, T* u_b, T* u_prev_b, T* u_next_b,    \
                     sgb_stream_t stream) {                                                    \
    return wave1d_gather<T>(n, D, c, c_b, u, u_b, u_prev_b, u_next_b, as_stream(stream));      \
  }                                                                                            \
  int wave1d_b_range_##SFX(int n, double D, T* c, T* c_b, T* u, T* u_b, T* u_prev_b,             \
                           T* u_next_b, long long j0, long long j1, sgb_stream_t stream) {      \
    if (j1 < 0) return einval("wave1d_b_range: bad range");                                    \
    return wave1d_gather<T>(n, D, c, c_b, u, u_b, u_prev_b, u_next_b, as_stream(stream), j0,   \
                            j1);                                                               \
  }                                                                                            \
  int wave1d_scatter_b_##SFX(int n, double D, T* c, T* c_b, T* u, T* u_b, T* u_prev_b,         \
                             T* u_next_b, sgb_stream_t stream) {                               \
    if (n <= 0 || !c || !c_b || !u || !u_b || !u_prev_b || !u_next_b)                          \
      return einval("wave1d_scatter_b: bad arguments");                                        \
    if (n < 3) return 0;                                                                       \
    wave1d_scatter_kernel<T><<<grid_1d(n - 2, 256), 256, 0, as_stream(stream)>>>(              \
        n, (T)D, c, c_b, u, u_b, u_prev_b, u_next_b);                                          \
    return launch_status("wave1d_scatter_b");                                                  \
  }
SGB_WAVE1D(double, f64)
SGB_WAVE1D(float, f32)

// ---- 3D stars
#define SGB_STAR3(NAME, MODE, T, SFX)                                                          \
  int NAME##_##SFX(int n, double D, T* c, T* u_1, T* u_2, T* u, sgb_stream_t stream) {         \
    return star3_primal<MODE, T>(#NAME, n, D, c, u_1, u_2, u, as_stream(stream));              \
  }                                                                                            \
  int NAME##_b_##SFX(int n, double D, T* c, T* c_b, T* u_1, T* u_1_b, T* u_2_b, T* u_b,        \
                     sgb_stream_t stream) {                                                    \
    return star3_gather<MODE, T>(#NAME "_b", n, D, c, c_b, u_1, u_1_b, u_2_b, u_b, 0, n, 0, n, \
                                 as_stream(stream));                                           \
  }                                                                                            \
  int NAME##_scatter_b_##SFX(int n, double D, T* c, T* c_b, T* u_1, T* u_1_b, T* u_2_b,        \
                             T* u_b, sgb_stream_t stream) {                                    \
    return star3_scatter<MODE, T>(#NAME "_scatter_b", n, D, c, c_b, u_1, u_1_b, u_2_b, u_b,    \
                                  as_stream(stream));                                          \
  }
SGB_STAR3(wave3d_c, 0, float, f32)
SGB_STAR3(wave3d_c, 0, double, f64)
SGB_STAR3(wave3d_c2, 1, float, f32)
SGB_STAR3(wave3d_c2, 1, double, f64)

#define SGB_R4(T, SFX)                                                                         \
  int wave3d_r4_##SFX(int n, double D, T* c, T* u_1, T* u_2, T* u, sgb_stream_t stream) {      \
    return star3_primal<2, T>("wave3d_r4", n, D, c, u_1, u_2, u, as_stream(stream));           \
  }                                                                                            \
  int wave3d_r4_b_##SFX(int n, double D, T* c, T* c_b, T* u_1, T* u_1_b, T* u_b,               \
                        sgb_stream_t stream) {                                                 \
    return star3_gather<2, T>("wave3d_r4_b", n, D, c, c_b, u_1, u_1_b, nullptr, u_b, 0, n, 0,  \
                              n, as_stream(stream));                                           \
  }                                                                                            \
  int wave3d_r4_scatter_b_##SFX(int n, double D, T* c, T* c_b, T* u_1, T* u_1_b, T* u_b,       \
                                sgb_stream_t stream) {                                         \
    return star3_scatter<2, T>("wave3d_r4_scatter_b", n, D, c, c_b, u_1, u_1_b, nullptr, u_b,  \
                               as_stream(stream));                                             \
  }
SGB_R4(float, f32)
SGB_R4(double, f64)

int wave3d_r4_b_slab_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                         float* u_b, int i_base, int nplanes, int out_i0, int out_i1,
                         sgb_stream_t stream) {
  return star3_gather<2, float>("wave3d_r4_b_slab", n, D, c, c_b, u_1, u_1_b, nullptr, u_b,
                                i_base, nplanes, out_i0, out_i1, as_stream(stream));
}

int wave3d_r4_b_fresh_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                              float* u_b, sgb_stream_t stream) {
  return r4_fresh("sgb_wave3d_r4_b_fresh", n, D, c, c_b, u_1, u_1_b, u_b, 0, n, 0, n,
                  as_stream(stream));
}

int wave3d_r4_b_fresh_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                          double* u_b, sgb_stream_t stream) {
  return r4_fresh("sgb_wave3d_r4_b_fresh_f64", n, D, c, c_b, u_1, u_1_b, u_b, 0, n, 0, n,
                  as_stream(stream));
}

int wave3d_r4_b_fresh_slab_f64(int n, double D, double* c, double* c_b, double* u_1,
                               double* u_1_b, double* u_b, int i_base, int nplanes, int out_i0,
                               int out_i1, sgb_stream_t stream) {
  return r4_fresh("sgb_wave3d_r4_b_fresh_slab_f64", n, D, c, c_b, u_1, u_1_b, u_b, i_base,
                  nplanes, out_i0, out_i1, as_stream(stream));
}

int wave3d_r4_b_fresh_slab_f32(int n, double D, float* c, float* c_b, float* u_1,
                                   float* u_1_b, float* u_b, int i_base, int nplanes,
                                   int out_i0, int out_i1, sgb_stream_t stream) {
  return r4_fresh("sgb_wave3d_r4_b_fresh_slab", n, D, c, c_b, u_1, u_1_b, u_b, i_base, nplanes,
                  out_i0, out_i1, as_stream(stream));
}

int wave3d_c_b_fresh_u2_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                            float* u_2_b, float* u_b, sgb_stream_t stream) {
  return star3_c_fresh_u2<0>("wave3d_c_b_fresh_u2", n, D, c, c_b, u_1, u_1_b, u_2_b, u_b,
                             as_stream(stream));
}

int wave3d_c2_b_fresh_u2_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                             float* u_2_b, float* u_b, sgb_stream_t stream) {
  return star3_c_fresh_u2<1>("wave3d_c2_b_fresh_u2", n, D, c, c_b, u_1, u_1_b, u_2_b, u_b,
                             as_stream(stream));
}

int sgb_wave3d_r4_b_step_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                             float* u_b, float* u_2_b, sgb_stream_t stream) {
  const char* name = "sgb_wave3d_r4_b_step";
  if (n <= 0) return einval(std::string(name) + ": n must be positive");
  if (!guard_ok(WAVE3D_R4, n)) return SGB_GUARD;
  if (!c || !c_b || !u_1 || !u_1_b || !u_b || !u_2_b)
    return einval(std::string(name) + ": null array");
  if (u_2_b == u_b || u_2_b == u_1_b || u_2_b == c_b)
    return einval(std::string(name) + ": u_2_b must not alias the other arrays");
  cudaStream_t s = as_stream(stream);
  if (star3_tma_ok<3, float>(n, {c, c_b, u_1, u_1_b, u_b, u_2_b}) &&
      !opt_flag(OPT_STEP_UNFUSED))
    return star3_v7_gather<3>(Slab3{n, 0, n}, 4, n - 5, 0, n, (float)D, c, c_b, u_1, u_1_b,
                              u_2_b, u_b, s, name);
  // other shapes: the two launches it fuses
  const int rc = wave3d_r4_b_f32(n, D, c, c_b, u_1, u_1_b, u_b, stream);
  if (rc != 0) return rc;
  return sgb_box_set_f32(u_2_b, u_b, -1.0, n, 4, n - 5, 0, n, stream);
}

int wave3d_r4_b_slab_peer_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                              float* u_b, int i_base, int nplanes, int out_i0, int out_i1,
                              const float* lo_c, const float* lo_u_1, const float* lo_u_b,
                              int lo_base, int lo_nplanes, const float* hi_c,
                              const float* hi_u_1, const float* hi_u_b, int hi_base,
                              int hi_nplanes, sgb_stream_t stream) {
  const char* name = "wave3d_r4_b_slab_peer";
  if (n <= 0 || nplanes <= 0) return einval(std::string(name) + ": bad sizes");
  if (!guard_ok(WAVE3D_R4, n)) return SGB_GUARD;
  if (!c || !c_b || !u_1 || !u_1_b || !u_b) return einval(std::string(name) + ": null array");
  if (!star3_tma_supported<2, float>(n))
    return einval(std::string(name) + ": needs n % 4 == 0 (TMA rows)");
  if (out_i1 == out_i0) return 0;
  const float* nc[2] = {lo_c, hi_c};
  const float* nu1[2] = {lo_u_1, hi_u_1};
  const float* nub[2] = {lo_u_b, hi_u_b};
  const int nb[2] = {lo_base, hi_base}, nn[2] = {lo_nplanes, hi_nplanes};
  return star3_v7_gather_peer<2>(Slab3{n, i_base, nplanes}, 4, n - 5, out_i0, out_i1, (float)D,
                                 c, c_b, u_1, u_1_b, u_b, nc, nu1, nub, nb, nn,
                                 as_stream(stream), name);
}

int sgb_ipc_handle(const void* ptr, void* handle64, long long* offset) {
  if (!ptr || !handle64 || !offset) return SGB_EINVAL;
  // allocation base of ptr (driver entry point, so the library keeps no hard
  // dependency on libcuda)
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  const GetRange get_range = reinterpret_cast<GetRange>(driver_entry("cuMemGetAddressRange"));
  CUdeviceptr base = 0;
  size_t size = 0;
  if (!get_range || get_range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
    return einval("sgb_ipc_handle: not a device allocation");
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
  if (e != cudaSuccess) return -static_cast<int>(e);
  std::memcpy(handle64, &h, sizeof(h));
  *offset = (long long)((CUdeviceptr)ptr - base);
  return 0;
}

int sgb_ipc_open(const void* handle64, long long offset, void** ptr) {
  if (!handle64 || !ptr) return SGB_EINVAL;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  const cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return -static_cast<int>(e);
  *ptr = (char*)base + offset;
  return 0;
}

int sgb_ipc_close(void* ptr, long long offset) {
  if (!ptr) return SGB_EINVAL;
  const cudaError_t e = cudaIpcCloseMemHandle((char*)ptr - offset);
  return e == cudaSuccess ? 0 : -static_cast<int>(e);
}

int wave3d_c_b_slab_f32(int n, double D, float* c, float* c_b, float* u_1, float* u_1_b,
                        float* u_2_b, float* u_b, int i_base, int nplanes, int out_i0,
                        int out_i1, sgb_stream_t stream) {
  return star3_gather<0, float>("wave3d_c_b_slab", n, D, c, c_b, u_1, u_1_b, u_2_b, u_b, i_base,
                                nplanes, out_i0, out_i1, as_stream(stream));
}

int wave3d_r4_b_slab_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                         double* u_b, int i_base, int nplanes, int out_i0, int out_i1,
                         sgb_stream_t stream) {
  return star3_gather<2, double>("wave3d_r4_b_slab", n, D, c, c_b, u_1, u_1_b, nullptr, u_b,
                                 i_base, nplanes, out_i0, out_i1, as_stream(stream));
}

int wave3d_c_b_slab_f64(int n, double D, double* c, double* c_b, double* u_1, double* u_1_b,
                        double* u_2_b, double* u_b, int i_base, int nplanes, int out_i0,
                        int out_i1, sgb_stream_t stream) {
  return star3_gather<0, double>("wave3d_c_b_slab", n, D, c, c_b, u_1, u_1_b, u_2_b, u_b,
                                 i_base, nplanes, out_i0, out_i1, as_stream(stream));
}

// ---- burgers2d
#define SGB_BURGERS(T, SFX)                                                                    \
  int burgers2d_##SFX(int n, double C, double D, T* u_1, T* u, sgb_stream_t stream) {          \
    if (n <= 0 || !u_1 || !u) return einval("burgers2d: bad arguments");                       \
    if (burgers2d_primal_ring<T>(n, C, D, u_1, u, as_stream(stream)))                          \
      return launch_status("burgers2d");                                                       \
    if (n % 2 == 0 && aligned16(u_1, u, u_1, u)) {                                             \
      dim3 g((unsigned)((n / 2 + 127) / 128), (unsigned)((n + 31) / 32));                      \
      burgers2d_primal_stream_kernel<T>                                                        \
          <<<g, 128, 0, as_stream(stream)>>>(n, (T)C, (T)D, u_1, u, 32);                       \
      return launch_status("burgers2d");                                                       \
    }                                                                                          \
    dim3 b(64, 4), g((unsigned)((n + 63) / 64), (unsigned)((n + 3) / 4));                      \
    burgers2d_primal_kernel<T><<<g, b, 0, as_stream(stream)>>>(n, (T)C, (T)D, u_1, u);         \
    return launch_status("burgers2d");                                                         \
  }                                                                                            \
  int burgers2d_b_##SFX(int n, double C, double D, T* u_1, T* u_1_b, T* u_b,                   \
                        sgb_stream_t stream) {                                                 \
    return burgers2d_gather<T>(n, C, D, u_1, u_1_b, u_b, as_stream(stream));                   \
  }                                                                                            \
  int burgers2d_b_rows_##SFX(int n, double C, double D, T* u_1, T* u_1_b, T* u_b, int row0,    \
                             int row1, sgb_stream_t stream) {                                  \
    return burgers2d_gather<T>(n, C, D, u_1, u_1_b, u_b, as_stream(stream), row0, row1);       \
  }                                                                                            \
  int burgers2d_scatter_b_##SFX(int n, double C, double D, T* u_1, T* u_1_b, T* u_b,           \
                                sgb_stream_t stream) {                                         \
    if (n <= 0 || !u_1 || !u_1_b || !u_b) return einval("burgers2d_scatter_b: bad arguments"); \
    if (n < 3) return 0;                                                                       \
    dim3 b(64, 4), g((unsigned)((n - 2 + 63) / 64), (unsigned)((n - 2 + 3) / 4));              \
    burgers2d_scatter_kernel<T><<<g, b, 0, as_stream(stream)>>>(n, (T)C, (T)D, u_1, u_1_b,     \
                                                                u_b);                          \
    return launch_status("burgers2d_scatter_b");                                               \
  }
SGB_BURGERS(double, f64)
SGB_BURGERS(float, f32)

}  // extern "C"
