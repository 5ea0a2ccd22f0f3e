// Streaming gather-adjoint kernels for the 1D wave (cfg 1) and 2D Burgers
// (cfg 3) families, fp64 or fp32.
//
// Same semantics as the per-point kernels in generic_kernels.cuh (the
// predicate form of the reference's hierarchical program, SURVEY Appendix C;
// partials of symdiff.cpp:238-305), restructured for HBM streaming:
//   * each thread owns 2 consecutive points (one 128-bit vector for fp64) so
//     every array element is loaded exactly once with a coalesced vector load;
//   * the k-1 / k+2 neighbours come from the adjacent lanes by warp shuffles
//     (only the two warp-edge lanes read an extra element, an L1 hit);
//   * burgers2d streams down the rows with a 3-row register queue of u_1 and
//     u_b, so rows are read once per row-chunk (plus one halo row per side).
#pragma once

#include "generic_kernels.cuh"

namespace sgb {

template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};

template <typename T>
__device__ __forceinline__ typename Vec2<T>::type ld2(const T* p) {
  return *reinterpret_cast<const typename Vec2<T>::type*>(p);
}
template <typename T>
__device__ __forceinline__ void st2(T* p, T a, T b) {
  typename Vec2<T>::type v;
  v.x = a;
  v.y = b;
  *reinterpret_cast<typename Vec2<T>::type*>(p) = v;
}

// value of lane-1's .y (left) / lane+1's .x (right); warp edges read memory
template <typename T>
__device__ __forceinline__ T left_of(T my_y, const T* row, long long j, long long n, int lane,
                                     bool active) {
  T v = __shfl_up_sync(0xffffffffu, my_y, 1);
  if (lane == 0) v = (active && j - 1 >= 0) ? row[j - 1] : T(0);
  return v;
}
template <typename T>
__device__ __forceinline__ T right_of(T my_x, const T* row, long long j, long long n, int lane,
                                      bool active) {
  T v = __shfl_down_sync(0xffffffffu, my_x, 1);
  if (lane == 31) v = (active && j + 2 < n) ? row[j + 2] : T(0);
  return v;
}

// ------------------------------------------------------------------ wave1d
template <typename T>
__global__ void __launch_bounds__(256) wave1d_stream_kernel(long long n, T D,
                                                            const T* __restrict__ c,
                                                            T* __restrict__ c_b,
                                                            const T* __restrict__ u,
                                                            T* __restrict__ u_b,
                                                            T* __restrict__ u_prev_b,
                                                            const T* __restrict__ s) {
  const int lane = threadIdx.x & 31;
  const long long j = 2 * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  const bool active = j < n;  // n even: both points or none
  const long long lo = 1, hi = n - 2;
  typename Vec2<T>::type cv{}, uv{}, sv{}, ob{}, op{}, ou{};
  if (active) {  // every load of this thread issued up front
    cv = ld2(c + j);
    uv = ld2(u + j);
    sv = ld2(s + j);
    ob = ld2(c_b + j);
    op = ld2(u_prev_b + j);
    ou = ld2(u_b + j);
  }
  // neighbours j-1 and j+2 of c, u, s (all warps participate in the shuffles)
  const T cl = left_of(cv.y, c, j, n, lane, active), cr = right_of(cv.x, c, j, n, lane, active);
  const T ul = left_of(uv.y, u, j, n, lane, active), ur = right_of(uv.x, u, j, n, lane, active);
  const T sl = left_of(sv.y, s, j, n, lane, active), sr = right_of(sv.x, s, j, n, lane, active);
  if (!active) return;
  // q = D c^2 s masked to the primal box at each of j-1 .. j+2
  auto q = [&](long long x, T cx, T sx) { return (x >= lo && x <= hi) ? D * cx * cx * sx : T(0); };
  const T q_l = q(j - 1, cl, sl), q0 = q(j, cv.x, sv.x), q1 = q(j + 1, cv.y, sv.y),
          q_r = q(j + 2, cr, sr);
  T out_ub[2], out_cb[2], out_pb[2];
  bool in[2], reach[2];
  const T cc[2] = {cv.x, cv.y}, uu[2] = {uv.x, uv.y}, ss[2] = {sv.x, sv.y};
  const T um[2] = {ul, uv.x}, up[2] = {uv.y, ur};  // u[y-1], u[y+1]
  const T qm[2] = {q_l, q0}, qc[2] = {q0, q1}, qp[2] = {q1, q_r};
#pragma unroll
  for (int m = 0; m < 2; m++) {
    const long long y = j + m;
    in[m] = y >= lo && y <= hi;
    reach[m] = y >= lo - 1 && y <= hi + 1;
    // terms: c@0, u@-1 (x=y+1), u@0, u@+1 (x=y-1), u_prev@0
    out_cb[m] = T(2) * D * (um[m] - T(2) * uu[m] + up[m]) * cc[m] * ss[m];
    out_ub[m] = qp[m] + (T(-2) * qc[m] + (in[m] ? T(2) * ss[m] : T(0))) + qm[m];
    out_pb[m] = -ss[m];
  }
  if (in[0] || in[1]) {
    st2(c_b + j, in[0] ? ob.x + out_cb[0] : ob.x, in[1] ? ob.y + out_cb[1] : ob.y);
    st2(u_prev_b + j, in[0] ? op.x + out_pb[0] : op.x, in[1] ? op.y + out_pb[1] : op.y);
  }
  if (reach[0] || reach[1])
    st2(u_b + j, reach[0] ? ou.x + out_ub[0] : ou.x, reach[1] ? ou.y + out_ub[1] : ou.y);
}

// ------------------------------------------------------------------ burgers2d
template <typename T>
__global__ void __launch_bounds__(128) burgers2d_stream_kernel(long long n, T C, T D,
                                                               const T* __restrict__ u1,
                                                               T* __restrict__ u1b,
                                                               const T* __restrict__ ub,
                                                               int rows_per_block) {
  const int lane = threadIdx.x & 31;
  const long long j = 2 * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  const bool active = j < n;
  const long long lo = 1, hi = n - 2;
  const long long i0 = (long long)blockIdx.y * rows_per_block;
  const long long i1 = min(i0 + rows_per_block, n);
  using V = typename Vec2<T>::type;
  auto row_u = [&](long long i) { return (active && i >= 0 && i < n) ? ld2(u1 + i * n + j) : V{}; };
  auto row_b = [&](long long i) { return (active && i >= 0 && i < n) ? ld2(ub + i * n + j) : V{}; };
  auto row_o = [&](long long i) { return (active && i >= 0 && i < n) ? ld2(u1b + i * n + j) : V{}; };
  V um = row_u(i0 - 1), u0 = row_u(i0), bm = row_b(i0 - 1), b0 = row_b(i0);
  V up = row_u(i0 + 1), bp = row_b(i0 + 1), o0 = row_o(i0);
  const bool jin[2] = {j >= lo && j <= hi, j + 1 >= lo && j + 1 <= hi};
  const bool jin_l = j - 1 >= lo && j - 1 <= hi, jin_r = j + 2 >= lo && j + 2 <= hi;
  for (long long i = i0; i < i1; i++) {
    // next iteration's rows are requested now (one row of lookahead)
    const V up2 = row_u(i + 2), bp2 = row_b(i + 2), o1 = row_o(i + 1);
    const T* urow = u1 + i * n;
    const T* brow = ub + i * n;
    const bool rowok = i >= 0 && i < n;
    const T ul = left_of(u0.y, urow, j, n, lane, active && rowok);
    const T ur = right_of(u0.x, urow, j, n, lane, active && rowok);
    const T bl = left_of(b0.y, brow, j, n, lane, active && rowok);
    const T br = right_of(b0.x, brow, j, n, lane, active && rowok);
    if (active) {
      const bool iin = i >= lo && i <= hi;
      const bool iin_m = i - 1 >= lo && i - 1 <= hi, iin_p = i + 1 >= lo && i + 1 <= hi;
      const T uc[2] = {u0.x, u0.y}, bc[2] = {b0.x, b0.y};
      const T uL[2] = {ul, u0.x}, uR[2] = {u0.y, ur};  // u[i][j-1], u[i][j+1]
      const T bL[2] = {bl, b0.x}, bR[2] = {b0.y, br};
      const bool jl[2] = {jin_l, jin[0]}, jr[2] = {jin[1], jin_r};
      const T uM[2] = {um.x, um.y}, uP[2] = {up.x, up.y}, bM[2] = {bm.x, bm.y},
              bP[2] = {bp.x, bp.y};
      T acc[2];
      bool reach[2];
#pragma unroll
      for (int m = 0; m < 2; m++) {
        // term order (symdiff.cpp:204): (-1,0), (0,-1), (0,0), (0,1), (1,0)
        T a = T(0);
        if (jin[m] && iin_p) a += burg_lower(C, D, uP[m]) * bP[m];
        if (iin && jr[m]) a += burg_lower(C, D, uR[m]) * bR[m];
        if (iin && jin[m]) a += burg_center(C, D, uc[m], uM[m], uP[m], uL[m], uR[m]) * bc[m];
        if (iin && jl[m]) a += burg_upper(C, D, uL[m]) * bL[m];
        if (jin[m] && iin_m) a += burg_upper(C, D, uM[m]) * bM[m];
        acc[m] = a;
        reach[m] = (iin && j + m >= lo - 1 && j + m <= hi + 1) ||
                   (jin[m] && i >= lo - 1 && i <= hi + 1);
      }
      if (reach[0] || reach[1])
        st2(u1b + i * n + j, reach[0] ? o0.x + acc[0] : o0.x, reach[1] ? o0.y + acc[1] : o0.y);
    }
    um = u0;
    u0 = up;
    up = up2;
    bm = b0;
    b0 = bp;
    bp = bp2;
    o0 = o1;
  }
}

}  // namespace sgb
