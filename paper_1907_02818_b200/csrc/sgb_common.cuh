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

inline unsigned grid_1d(long long work, int block) {
  long long g = (work + block - 1) / block;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace sgb
