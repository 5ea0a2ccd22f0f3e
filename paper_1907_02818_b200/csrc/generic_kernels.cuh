// Per-point kernels for every family: primal, gather adjoint (predicate form
// of the hierarchical core+boundary program) and the atomic scatter ablation.
//
// These are the general-shape path (any n, fp32 or fp64, slab or full grid).
// The streaming TMA kernel in star3d_tma.cuh replaces the gather adjoint for
// 3D stars when the shape allows it.
//
// Semantics follow SURVEY Appendix C, derived from the reference:
//   gather  : for y in the write box, for l ascending with y - o_l in B:
//             adj_l[y] += S_l(y - o_l) * seed[y - o_l]          (interp.cpp:189-198)
//   scatter : for x in B, l ascending: adj_l[x + o_l] += S_l(x) * seed[x]
//                                                              (interp.cpp:200-228)
// with the partials S_l of symdiff.cpp:238-305 for each spec in oracle/specs.
#pragma once

#include "sgb_common.cuh"

namespace sgb {

// ------------------------------------------------------------------ 3D stars
// MODE 0: wave3d_c  (c linear; u_2 active)
// MODE 1: wave3d_c2 (c^2;      u_2 active)
// MODE 2: wave3d_r4 (c^2;      u_2 passive; radius 4)
// MODE 3: wave3d_r4 gather that also writes the u_2 partial of a time loop,
//         u_2_b = -u_b on B and 0 elsewhere (drivers.time_loop_adjoint; the
//         fused form of gather + sgb_box_set, fp32 streaming kernel only)
// MODE 4: wave3d_r4 gather whose u_1_b is this step's adjoint alone (u_1_b =
//         0 + sum where reached, 0 elsewhere: the fused form of zeroing u_1_b
//         and accumulating, cfg 5's independent steps; fp32 streaming only)
template <int MODE>
struct Star3 {
  static constexpr int R = MODE >= 2 ? 4 : 1;
  static constexpr bool kU2 = MODE < 2;
  static constexpr bool kU2Set = MODE == 3;
  static constexpr bool kU1bFresh = MODE == 4;
  static constexpr bool kC2 = MODE != 0;
  static constexpr bool kIncrement = MODE != 2;  // primal mode of the spec
  // weight of offset |r| along one axis; r == 0 gives the folded 3-axis centre
  template <typename T>
  __device__ __forceinline__ static T w(int r) {
    if (R == 1) return r == 0 ? T(-6) : T(1);
    return r == 0 ? T(kW4C3) : T(w4(r));
  }
};

// Slab-aware grid view: local planes [i_base, i_base + nplanes) of an n^3 grid.
struct Slab3 {
  long long n, i_base, nplanes;
  __device__ __forceinline__ long long idx(long long gi, long long j, long long k) const {
    return ((gi - i_base) * n + j) * n + k;
  }
};

template <int MODE, typename T>
__device__ __forceinline__ T star_lap(const T* __restrict__ u, const Slab3& g, long long i,
                                      long long j, long long k) {
  using S = Star3<MODE>;
  T s = S::template w<T>(0) * u[g.idx(i, j, k)];
#pragma unroll
  for (int r = 1; r <= S::R; r++)
    s += S::template w<T>(r) * (u[g.idx(i - r, j, k)] + u[g.idx(i + r, j, k)] +
                                 u[g.idx(i, j - r, k)] + u[g.idx(i, j + r, k)] +
                                 u[g.idx(i, j, k - r)] + u[g.idx(i, j, k + r)]);
  return s;
}

template <int MODE, typename T>
__global__ void star3_primal_kernel(Slab3 g, long long lo, long long hi, long long out_i0,
                                    long long out_i1, T D, const T* __restrict__ c,
                                    const T* __restrict__ u_1, const T* __restrict__ u_2,
                                    T* __restrict__ u) {
  using S = Star3<MODE>;
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long j = blockIdx.y * (long long)blockDim.y + threadIdx.y;
  const long long i = out_i0 + blockIdx.z;
  if (i >= out_i1 || k < lo || k > hi || j < lo || j > hi || i < lo || i > hi) return;
  const long long x = g.idx(i, j, k);
  const T cc = S::kC2 ? c[x] * c[x] : c[x];
  const T v = T(2) * u_1[x] - u_2[x] + cc * D * star_lap<MODE>(u_1, g, i, j, k);
  if (S::kIncrement)
    u[x] += v;
  else
    u[x] = v;
}

template <int MODE, typename T>
__global__ void star3_gather_kernel(Slab3 g, long long lo, long long hi, long long out_i0,
                                    long long out_i1, T D, const T* __restrict__ c,
                                    T* __restrict__ c_b, const T* __restrict__ u_1,
                                    T* __restrict__ u_1_b, T* __restrict__ u_2_b,
                                    const T* __restrict__ u_b) {
  using S = Star3<MODE>;
  constexpr int R = S::R;
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long j = blockIdx.y * (long long)blockDim.y + threadIdx.y;
  const long long i = out_i0 + blockIdx.z;
  const long long n = g.n;
  if (i >= out_i1 || k >= n || j >= n) return;
  if (!star_reached<R>(i, j, k, lo, hi)) return;  // no valid term: untouched
  const bool inB = in_range(i, lo, hi) && in_range(j, lo, hi) && in_range(k, lo, hi);
  auto q = [&](long long a, long long b, long long e) -> T {  // coef(c) * seed at x, masked
    if (!(in_range(a, lo, hi) && in_range(b, lo, hi) && in_range(e, lo, hi))) return T(0);
    const long long x = g.idx(a, b, e);
    const T cc = S::kC2 ? c[x] * c[x] : c[x];
    return D * cc * u_b[x];
  };
  T acc = T(0);
#pragma unroll
  for (int r = 1; r <= R; r++)
    acc += S::template w<T>(r) * (q(i + r, j, k) + q(i - r, j, k) + q(i, j + r, k) +
                                  q(i, j - r, k) + q(i, j, k + r) + q(i, j, k - r));
  const long long y = g.idx(i, j, k);
  if (inB) {
    const T ub = u_b[y];
    acc += S::template w<T>(0) * q(i, j, k) + T(2) * ub;
    const T lap = star_lap<MODE>(u_1, g, i, j, k);
    const T sc = S::kC2 ? T(2) * D * c[y] : D;  // S_c = sc * Lap
    c_b[y] += sc * lap * ub;
    if (S::kU2) u_2_b[y] += -ub;
  }
  u_1_b[y] += acc;
}

template <int MODE, typename T>
__global__ void star3_scatter_kernel(Slab3 g, long long lo, long long hi, T D,
                                     const T* __restrict__ c, T* __restrict__ c_b,
                                     const T* __restrict__ u_1, T* __restrict__ u_1_b,
                                     T* __restrict__ u_2_b, const T* __restrict__ u_b) {
  using S = Star3<MODE>;
  constexpr int R = S::R;
  const long long k = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long j = lo + blockIdx.y * (long long)blockDim.y + threadIdx.y;
  const long long i = lo + blockIdx.z;
  if (k > hi || j > hi) return;
  const long long x = g.idx(i, j, k);
  const T sd = u_b[x];
  const T cv = c[x];
  const T cc = S::kC2 ? cv * cv : cv;
  // term order: c, then u_1 offsets lexicographic, then u_2 (symdiff.cpp:204-223)
  const T sc = S::kC2 ? T(2) * D * cv : D;
  atomicAdd(&c_b[x], sc * star_lap<MODE>(u_1, g, i, j, k) * sd);
  const T cu = D * cc * sd;
#pragma unroll
  for (int r = R; r >= 1; r--) atomicAdd(&u_1_b[g.idx(i - r, j, k)], S::template w<T>(r) * cu);
#pragma unroll
  for (int r = R; r >= 1; r--) atomicAdd(&u_1_b[g.idx(i, j - r, k)], S::template w<T>(r) * cu);
#pragma unroll
  for (int r = R; r >= 1; r--) atomicAdd(&u_1_b[g.idx(i, j, k - r)], S::template w<T>(r) * cu);
  atomicAdd(&u_1_b[x], (S::template w<T>(0) * D * cc + T(2)) * sd);
#pragma unroll
  for (int r = 1; r <= R; r++) atomicAdd(&u_1_b[g.idx(i, j, k + r)], S::template w<T>(r) * cu);
#pragma unroll
  for (int r = 1; r <= R; r++) atomicAdd(&u_1_b[g.idx(i, j + r, k)], S::template w<T>(r) * cu);
#pragma unroll
  for (int r = 1; r <= R; r++) atomicAdd(&u_1_b[g.idx(i + r, j, k)], S::template w<T>(r) * cu);
  if (S::kU2) atomicAdd(&u_2_b[x], -sd);
}

// ------------------------------------------------------------------ wave1d
template <typename T>
__global__ void wave1d_primal_kernel(long long n, T D, const T* __restrict__ c,
                                     const T* __restrict__ u, const T* __restrict__ u_prev,
                                     T* __restrict__ u_next) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < 1 || i > n - 2) return;
  const T ui = u[i];
  u_next[i] = T(2) * ui - u_prev[i] + c[i] * c[i] * D * (u[i - 1] - T(2) * ui + u[i + 1]);
}

template <typename T>
__global__ void wave1d_gather_kernel(long long n, T D, const T* __restrict__ c,
                                     T* __restrict__ c_b, const T* __restrict__ u,
                                     T* __restrict__ u_b, T* __restrict__ u_prev_b,
                                     const T* __restrict__ s) {
  const long long y = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long lo = 1, hi = n - 2;
  if (y >= n) return;
  T acc = T(0);
  if (y + 1 >= lo && y + 1 <= hi) acc += D * c[y + 1] * c[y + 1] * s[y + 1];  // o = -1
  if (y >= lo && y <= hi) {
    const T cy = c[y], sy = s[y];
    c_b[y] += T(2) * D * (u[y - 1] - T(2) * u[y] + u[y + 1]) * cy * sy;   // o = 0 (c)
    acc += (T(-2) * D * cy * cy + T(2)) * sy;                              // o = 0 (u)
    u_prev_b[y] += -sy;                                                    // u_prev
  }
  if (y - 1 >= lo && y - 1 <= hi) acc += D * c[y - 1] * c[y - 1] * s[y - 1];  // o = +1
  if (y >= lo - 1 && y <= hi + 1) u_b[y] += acc;
}

template <typename T>
__global__ void wave1d_scatter_kernel(long long n, T D, const T* __restrict__ c,
                                      T* __restrict__ c_b, const T* __restrict__ u,
                                      T* __restrict__ u_b, T* __restrict__ u_prev_b,
                                      const T* __restrict__ s) {
  const long long x = 1 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (x > n - 2) return;
  const T cx = c[x], sx = s[x];
  atomicAdd(&c_b[x], T(2) * D * (u[x - 1] - T(2) * u[x] + u[x + 1]) * cx * sx);
  atomicAdd(&u_b[x - 1], D * cx * cx * sx);
  atomicAdd(&u_b[x], (T(-2) * D * cx * cx + T(2)) * sx);
  atomicAdd(&u_b[x + 1], D * cx * cx * sx);
  atomicAdd(&u_prev_b[x], -sx);
}

// ------------------------------------------------------------------ burgers2d
template <typename T>
__device__ __forceinline__ T sel_ge0(T v) { return v >= T(0) ? T(1) : T(0); }

// S for o = (-1,0) / (0,-1) at x
template <typename T>
__device__ __forceinline__ T burg_lower(T C, T D, T u) { return C * fmax(T(0), u) + D; }
// S for o = (0,1) / (1,0) at x
template <typename T>
__device__ __forceinline__ T burg_upper(T C, T D, T u) { return -C * fmin(T(0), u) + D; }
// S for o = (0,0) at x (symdiff.cpp:269-274 select rules)
template <typename T>
__device__ __forceinline__ T burg_center(T C, T D, T u, T um, T up, T vm, T vp) {
  const T ge = sel_ge0(u), le = sel_ge0(-u);
  return -C * ((u - um) * ge + (u - vm) * ge + (vp - u) * le + (up - u) * le +
               T(2) * fmax(T(0), u) - T(2) * fmin(T(0), u)) -
         T(4) * D + T(1);
}

template <typename T>
__global__ void burgers2d_primal_kernel(long long n, T C, T D, const T* __restrict__ u1,
                                        T* __restrict__ u) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long i = blockIdx.y * (long long)blockDim.y + threadIdx.y;
  if (i < 1 || i > n - 2 || j < 1 || j > n - 2) return;
  const long long x = i * n + j;
  const T v = u1[x], um = u1[x - n], up = u1[x + n], vm = u1[x - 1], vp = u1[x + 1];
  u[x] = v -
         C * (fmax(v, T(0)) * (v - um) + fmin(v, T(0)) * (up - v) + fmax(v, T(0)) * (v - vm) +
              fmin(v, T(0)) * (vp - v)) +
         D * (up + um + vp + vm - T(4) * v);
}

template <typename T>
__global__ void burgers2d_gather_kernel(long long n, T C, T D, const T* __restrict__ u1,
                                        T* __restrict__ u1_b, const T* __restrict__ ub) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long i = blockIdx.y * (long long)blockDim.y + threadIdx.y;
  const long long lo = 1, hi = n - 2;
  if (i >= n || j >= n) return;
  const bool iin = in_range(i, lo, hi), jin = in_range(j, lo, hi);
  if (!((iin && j >= lo - 1 && j <= hi + 1) || (jin && i >= lo - 1 && i <= hi + 1))) return;
  const long long y = i * n + j;
  T acc = T(0);
  if (jin && in_range(i + 1, lo, hi)) acc += burg_lower(C, D, u1[y + n]) * ub[y + n];
  if (iin && in_range(j + 1, lo, hi)) acc += burg_lower(C, D, u1[y + 1]) * ub[y + 1];
  if (iin && jin)
    acc += burg_center(C, D, u1[y], u1[y - n], u1[y + n], u1[y - 1], u1[y + 1]) * ub[y];
  if (iin && in_range(j - 1, lo, hi)) acc += burg_upper(C, D, u1[y - 1]) * ub[y - 1];
  if (jin && in_range(i - 1, lo, hi)) acc += burg_upper(C, D, u1[y - n]) * ub[y - n];
  u1_b[y] += acc;
}

template <typename T>
__global__ void burgers2d_scatter_kernel(long long n, T C, T D, const T* __restrict__ u1,
                                         T* __restrict__ u1_b, const T* __restrict__ ub) {
  const long long j = 1 + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long i = 1 + blockIdx.y * (long long)blockDim.y + threadIdx.y;
  if (i > n - 2 || j > n - 2) return;
  const long long x = i * n + j;
  const T u = u1[x], sd = ub[x];
  atomicAdd(&u1_b[x - n], burg_lower(C, D, u) * sd);
  atomicAdd(&u1_b[x - 1], burg_lower(C, D, u) * sd);
  atomicAdd(&u1_b[x], burg_center(C, D, u, u1[x - n], u1[x + n], u1[x - 1], u1[x + 1]) * sd);
  atomicAdd(&u1_b[x + 1], burg_upper(C, D, u) * sd);
  atomicAdd(&u1_b[x + n], burg_upper(C, D, u) * sd);
}

}  // namespace sgb
