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
#include "star3d_tma.cuh"

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
                                                            const T* __restrict__ s,
                                                            long long j0, long long j1) {
  // outputs j in [j0, j1) (j0 even; the full grid: 0, n); inputs are read at
  // j-1 .. j+2, so [j0-1, j1] must be resident
  const int lane = threadIdx.x & 31;
  const long long j = j0 + 2 * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  const bool active = j < j1;   // n, j0, j1 even: both points or none
  const bool inside = j < n;    // lanes past j1 still feed their neighbours' shuffles
  const long long lo = 1, hi = n - 2;
  typename Vec2<T>::type cv{}, uv{}, sv{}, ob{}, op{}, ou{};
  if (inside) {  // every input load of this thread issued up front
    cv = ld2(c + j);
    uv = ld2(u + j);
    sv = ld2(s + j);
  }
  if (active) {
    ob = ld2(c_b + j);
    op = ld2(u_prev_b + j);
    ou = ld2(u_b + j);
  }
  // neighbours j-1 and j+2 of c, u, s (all warps participate in the shuffles)
  const T cl = left_of(cv.y, c, j, n, lane, inside), cr = right_of(cv.x, c, j, n, lane, inside);
  const T ul = left_of(uv.y, u, j, n, lane, inside), ur = right_of(uv.x, u, j, n, lane, inside);
  const T sl = left_of(sv.y, s, j, n, lane, inside), sr = right_of(sv.x, s, j, n, lane, inside);
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

// ------------------------------------------------------------------ burgers2d primal
// run_nest of the Burgers spec on [1, n-2]^2 (interp.cpp:153-173): each thread
// owns 2 consecutive j of a column strip and streams down rows_per_block
// rows with a 3-row register window (row i+1 requested one row ahead);
// j-1 / j+2 from the neighbouring lanes.  Same expression and grouping as
// the per-point kernel (generic_kernels.cuh).  16 B/pt: u_1 read, u written.
template <typename T>
__global__ void __launch_bounds__(128) burgers2d_primal_stream_kernel(long long n, T C, T D,
                                                                      const T* __restrict__ u1,
                                                                      T* __restrict__ u,
                                                                      int rows_per_block) {
  using V = typename Vec2<T>::type;
  const int lane = threadIdx.x & 31;
  const long long j = 2 * (blockIdx.x * (long long)blockDim.x + threadIdx.x);
  const bool active = j < n;
  const long long i0 = (long long)blockIdx.y * rows_per_block;
  const long long i1 = min(i0 + rows_per_block, n);
  auto row = [&](long long i) { return (active && i >= 0 && i < n) ? ld2(u1 + i * n + j) : V{}; };
  V um = row(i0 - 1), u0 = row(i0), up = row(i0 + 1);
  const bool jin[2] = {j >= 1 && j <= n - 2, j + 1 >= 1 && j + 1 <= n - 2};
  for (long long i = i0; i < i1; i++) {
    const V up2 = row(i + 2);
    const T* urow = u1 + i * n;
    const bool rowok = i >= 0 && i < n;
    const T ul = left_of(u0.y, urow, j, n, lane, active && rowok);
    const T ur = right_of(u0.x, urow, j, n, lane, active && rowok);
    if (active && i >= 1 && i <= n - 2 && (jin[0] || jin[1])) {
      const T vv[2] = {u0.x, u0.y}, mm[2] = {um.x, um.y}, pp[2] = {up.x, up.y};
      const T vl[2] = {ul, u0.x}, vr[2] = {u0.y, ur};
      T out[2];
#pragma unroll
      for (int m = 0; m < 2; m++) {
        const T v = vv[m];
        out[m] = v -
                 C * (fmax(v, T(0)) * (v - mm[m]) + fmin(v, T(0)) * (pp[m] - v) +
                      fmax(v, T(0)) * (v - vl[m]) + fmin(v, T(0)) * (vr[m] - v)) +
                 D * (pp[m] + mm[m] + vr[m] + vl[m] - T(4) * v);
      }
      T* orow = u + i * n + j;
      if (jin[0] && jin[1]) {
        st2(orow, out[0], out[1]);
      } else {
        if (jin[0]) orow[0] = out[0];
        if (jin[1]) orow[1] = out[1];
      }
    }
    um = u0;
    u0 = up;
    up = up2;
  }
}

// ------------------------------------------------------------------ burgers2d (ring)
// Strip-streaming form: a CTA owns a W-column strip and rows [i0, i1).  One
// thread streams the row segments of u_1 and u_b (with a 16-byte halo each
// side) and of u_1_b into an S-stage shared-memory ring with 1D bulk copies
// (cp.async.bulk, mbarrier complete_tx), S-3 rows ahead of the consumers, so
// memory-level parallelism no longer depends on registers or occupancy.
// Every thread then evaluates its two points from shared memory (no shuffles,
// no 64-bit index math in the loop); term order and predicates as above.
namespace tma {
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace tma

template <typename T, int S_ = 4>
struct BurgRing {
  static constexpr int THREADS = 128, W = 2 * THREADS;  // strip width (columns)
  static constexpr int H = 16 / (int)sizeof(T);          // halo columns: one 16-B granule
  static constexpr int UW = W + 2 * H;                   // u_1 / u_b row segment
  static constexpr int S = S_;                           // ring stages (rows)
  static constexpr int STAGE = 2 * UW + W;               // u_1, u_b, u_1_b (elements)
  static constexpr int SMEM = S * STAGE * (int)sizeof(T) + S * 8;
};

template <typename T>
__device__ __forceinline__ void st2cs(T* p, T a, T b) {
  typename Vec2<T>::type v;
  v.x = a;
  v.y = b;
  __stcs(reinterpret_cast<typename Vec2<T>::type*>(p), v);
}
// max(0, u) / min(0, u) as one compare + select: equal to fmax / fmin for
// every u up to the sign of a zero result (absorbed by the + D / the sums
// they enter), and for NaN u (both give 0)
template <typename T>
__device__ __forceinline__ T pos0(T u) { return u > T(0) ? u : T(0); }
template <typename T>
__device__ __forceinline__ T neg0(T u) { return u < T(0) ? u : T(0); }

// Strip-streaming form: a CTA owns a W-column strip and rows [i0, i1).  One
// thread streams the row segments of u_1 and u_b (with a 16-byte halo each
// side) and of u_1_b into an S-stage shared-memory ring with 1D bulk copies
// (cp.async.bulk, mbarrier complete_tx), S-3 rows ahead of the consumers;
// stages are small (6 KB fp64) so 8 CTAs (32 warps) stay resident per SM.
// Every thread evaluates its two points from shared memory (no shuffles, no
// 64-bit index math in the loop) in the reference's term order
// (symdiff.cpp:204): (-1,0), (0,-1), (0,0), (0,1), (1,0).
template <typename T, int S_>
__global__ void __launch_bounds__(BurgRing<T, S_>::THREADS, 8)
    burgers2d_ring_kernel(int n, T C, T D, const T* __restrict__ u1, T* __restrict__ u1b,
                          const T* __restrict__ ub, int rows_per_block, int row_lo,
                          int row_hi) {
  // output rows [row_lo, row_hi) (the full grid: 0, n); rows row_lo-1 ..
  // row_hi of u_1 / u_b must be resident
  using Rg = BurgRing<T, S_>;
  using V = typename Vec2<T>::type;
  constexpr int W = Rg::W, H = Rg::H, UW = Rg::UW, S = Rg::S, ST = Rg::STAGE;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + S * ST);
  const int tid = threadIdx.x;
  const int j0 = blockIdx.x * W;
  const int i0 = row_lo + blockIdx.y * rows_per_block;
  const int i1 = min(i0 + rows_per_block, row_hi);
  const int lo = 1, hi = n - 2;
  const int ca = max(j0 - H, 0), cb = min(j0 + W + H, n), oa = j0, ob = min(j0 + W, n);
  const uint32_t ubytes = (uint32_t)(cb - ca) * sizeof(T), obytes = (uint32_t)(ob - oa) * sizeof(T);
  const int uoff = ca - (j0 - H);
  const int r_first = i0 - 1, nrows = i1 - i0 + 2;  // rows i0-1 .. i1

  for (int e = tid; e < S * ST; e += Rg::THREADS) ring[e] = T(0);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros before bulk writes
  __syncthreads();

  auto issue = [&](int k) {
    const int s = k % S, r = r_first + k;
    T* st = ring + s * ST;
    const bool valid = r >= 0 && r < n, own = r >= i0 && r < i1;
    tma::mbar_arrive_expect_tx(&bars[s], valid ? 2 * ubytes + (own ? obytes : 0u) : 0u);
    if (valid) {
      const size_t rb = (size_t)r * n;
      tma::bulk_g2s(st + uoff, u1 + rb + ca, ubytes, &bars[s]);
      tma::bulk_g2s(st + UW + uoff, ub + rb + ca, ubytes, &bars[s]);
      if (own) tma::bulk_g2s(st + 2 * UW, u1b + rb + oa, obytes, &bars[s]);
    }
  };
  if (tid == 0)
    for (int k = 0; k < S && k < nrows; k++) issue(k);

  const int jl = 2 * tid, j = j0 + jl;
  const bool active = j < n;
  auto inB = [&](int x) { return x >= lo && x <= hi; };
  const bool jin[2] = {inB(j), inB(j + 1)};
  const bool jl_[2] = {inB(j - 1), jin[0]}, jr_[2] = {jin[1], inB(j + 2)};
  const bool jreach[2] = {j >= lo - 1 && j <= hi + 1, j + 1 >= lo - 1 && j + 1 <= hi + 1};
  // columns j, j+1 and their k-neighbours all inside [lo, hi]
  const bool inner = jl_[0] && jin[0] && jin[1] && jr_[1];
  T* orow = u1b + (size_t)i0 * n + j;
  tma::mbar_wait(&bars[0], 0);
  // stages of rows r-1, r, r+1 (row r is ring row k = r - r_first) and the
  // parities of the latter two, advanced incrementally (no k % S per row)
  int sm = 0, sc = 1 % S, sp = 2 % S;
  uint32_t phc = 0, php = S > 2 ? 0u : 1u;
  for (int r = i0; r < i1; r++, orow += n) {
    const int k = r - r_first;
    tma::mbar_wait(&bars[sc], phc);
    tma::mbar_wait(&bars[sp], php);
    if (active) {
      const T* Um = ring + sm * ST + H + jl;
      const T* Uc = ring + sc * ST + H + jl;
      const T* Up = ring + sp * ST + H + jl;
      const V um = *reinterpret_cast<const V*>(Um), uc = *reinterpret_cast<const V*>(Uc),
              up = *reinterpret_cast<const V*>(Up);
      const V bm = *reinterpret_cast<const V*>(Um + UW), bc = *reinterpret_cast<const V*>(Uc + UW),
              bp = *reinterpret_cast<const V*>(Up + UW);
      const V oc = *reinterpret_cast<const V*>(Uc - H + 2 * UW);  // u_1_b at (r, j)
      const T ul = Uc[-1], ur = Uc[2], bl = Uc[UW - 1], br = Uc[UW + 2];
      const bool iin = inB(r), iin_m = inB(r - 1), iin_p = inB(r + 1);
      const bool ireach = r >= lo - 1 && r <= hi + 1;
      const T ucv[2] = {uc.x, uc.y}, bcv[2] = {bc.x, bc.y};
      const T uL[2] = {ul, uc.x}, uR[2] = {uc.y, ur};
      const T bL[2] = {bl, bc.x}, bR[2] = {bc.y, br};
      const T uM[2] = {um.x, um.y}, uP[2] = {up.x, up.y}, bM[2] = {bm.x, bm.y},
              bP[2] = {bp.x, bp.y};
      T acc[2];
      bool reach[2];
      auto terms = [&](int m, T& t1, T& t2, T& tc, T& t4, T& t5) {
        const T u = ucv[m];
        const T ge = u >= T(0) ? T(1) : T(0), le = -u >= T(0) ? T(1) : T(0);
        const T cen = -C * ((u - uM[m]) * ge + (u - uL[m]) * ge + (uR[m] - u) * le +
                            (uP[m] - u) * le + T(2) * pos0(u) - T(2) * neg0(u)) -
                      T(4) * D + T(1);
        t1 = (C * pos0(uP[m]) + D) * bP[m];
        t2 = (C * pos0(uR[m]) + D) * bR[m];
        tc = cen * bcv[m];
        t4 = (-C * neg0(uL[m]) + D) * bL[m];
        t5 = (-C * neg0(uM[m]) + D) * bM[m];
      };
      if (iin && iin_m && iin_p && inner) {
        // both points and all five terms inside the box (all but a 2-point
        // frame): the same sums without the per-term masks
#pragma unroll
        for (int m = 0; m < 2; m++) {
          T t1, t2, tc, t4, t5;
          terms(m, t1, t2, tc, t4, t5);
          T a = T(0) + t1;
          a += t2;
          a += tc;
          a += t4;
          a += t5;
          acc[m] = a;
        }
        st2cs(orow, oc.x + acc[0], oc.y + acc[1]);
      } else {
#pragma unroll
        for (int m = 0; m < 2; m++) {
          T t1, t2, tc, t4, t5;
          terms(m, t1, t2, tc, t4, t5);
          T a = T(0);
          a += jin[m] && iin_p ? t1 : T(0);
          a += iin && jr_[m] ? t2 : T(0);
          a += iin && jin[m] ? tc : T(0);
          a += iin && jl_[m] ? t4 : T(0);
          a += jin[m] && iin_m ? t5 : T(0);
          acc[m] = a;
          reach[m] = (iin && jreach[m]) || (jin[m] && ireach);
        }
        if (reach[0] || reach[1])
          st2cs(orow, reach[0] ? oc.x + acc[0] : oc.x, reach[1] ? oc.y + acc[1] : oc.y);
      }
    }
    __syncthreads();  // row r-1's stage is free
    if (tid == 0 && k - 1 + S < nrows) issue(k - 1 + S);
    sm = sc;
    sc = sp;
    phc = php;
    if (++sp == S) sp = 0, php ^= 1u;
  }
}

// ------------------------------------------------------------------ burgers2d primal (ring)
// The primal in the strip-streaming form of the adjoint ring kernel: one
// thread streams the u_1 row segments (W columns + a 16-byte halo each side)
// of rows i0-1 .. i1 into an S-stage ring with 1D bulk copies, S-3 rows
// ahead; every thread evaluates its two points of row r from shared memory
// (rows r-1, r, r+1) with the same expression and grouping as
// burgers2d_primal_stream_kernel / the per-point kernel (bitwise equal).
// The register-streaming form it replaces was issue-bound on row-index math
// and waited on its own loads (profiles/).  16 B/pt: u_1 read, u written.
template <typename T, int S_>
struct BurgPrimalRing {
  static constexpr int THREADS = 128, W = 2 * THREADS;
  static constexpr int H = 16 / (int)sizeof(T);
  static constexpr int UW = W + 2 * H;
  static constexpr int S = S_;
  static constexpr int SMEM = S * UW * (int)sizeof(T) + S * 8;
};

template <typename T, int S_>
__global__ void __launch_bounds__(128, 8)
    burgers2d_primal_ring_kernel(int n, T C, T D, const T* __restrict__ u1, T* __restrict__ u,
                                 int rows_per_block) {
  using Rg = BurgPrimalRing<T, S_>;
  using V = typename Vec2<T>::type;
  constexpr int W = Rg::W, H = Rg::H, UW = Rg::UW, S = Rg::S;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* ring = reinterpret_cast<T*>(smem_raw);
  uint64_t* bars = reinterpret_cast<uint64_t*>(ring + S * UW);
  const int tid = threadIdx.x;
  const int j0 = blockIdx.x * W;
  const int i0 = blockIdx.y * rows_per_block;
  const int i1 = min(i0 + rows_per_block, n);
  const int ca = max(j0 - H, 0), cb = min(j0 + W + H, n);
  const uint32_t ubytes = (uint32_t)(cb - ca) * sizeof(T);
  const int uoff = ca - (j0 - H);
  const int r_first = i0 - 1, nrows = i1 - i0 + 2;  // rows i0-1 .. i1

  // columns outside the grid are never loaded: zero once (never read for an
  // output point either, the outputs are j in [1, n-2])
  for (int e = tid; e < S * UW; e += Rg::THREADS) ring[e] = T(0);
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < S; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();

  auto issue = [&](int k) {
    const int s = k % S, r = r_first + k;
    const bool valid = r >= 0 && r < n;
    tma::mbar_arrive_expect_tx(&bars[s], valid ? ubytes : 0u);
    if (valid) tma::bulk_g2s(ring + s * UW + uoff, u1 + (size_t)r * n + ca, ubytes, &bars[s]);
  };
  if (tid == 0)
    for (int k = 0; k < S && k < nrows; k++) issue(k);

  const int jl = 2 * tid, j = j0 + jl;
  const bool active = j < n;
  const bool jin[2] = {j >= 1 && j <= n - 2, j + 1 >= 1 && j + 1 <= n - 2};
  T* orow = u + (size_t)i0 * n + j;
  tma::mbar_wait(&bars[0], 0);
  int sm = 0, sc = 1 % S, sp = 2 % S;  // as in burgers2d_ring_kernel
  uint32_t phc = 0, php = S > 2 ? 0u : 1u;
  for (int r = i0; r < i1; r++, orow += n) {
    const int k = r - r_first;
    tma::mbar_wait(&bars[sc], phc);
    tma::mbar_wait(&bars[sp], php);
    if (active && r >= 1 && r <= n - 2 && (jin[0] || jin[1])) {
      const T* Um = ring + sm * UW + H + jl;
      const T* Uc = ring + sc * UW + H + jl;
      const T* Up = ring + sp * UW + H + jl;
      const V um = *reinterpret_cast<const V*>(Um), u0 = *reinterpret_cast<const V*>(Uc),
              up = *reinterpret_cast<const V*>(Up);
      const T ul = Uc[-1], ur = Uc[2];
      const T vv[2] = {u0.x, u0.y}, mm[2] = {um.x, um.y}, pp[2] = {up.x, up.y};
      const T vl[2] = {ul, u0.x}, vr[2] = {u0.y, ur};
      T out[2];
#pragma unroll
      for (int m = 0; m < 2; m++) {
        const T v = vv[m];
        out[m] = v -
                 C * (fmax(v, T(0)) * (v - mm[m]) + fmin(v, T(0)) * (pp[m] - v) +
                      fmax(v, T(0)) * (v - vl[m]) + fmin(v, T(0)) * (vr[m] - v)) +
                 D * (pp[m] + mm[m] + vr[m] + vl[m] - T(4) * v);
      }
      if (jin[0] && jin[1]) {
        st2cs(orow, out[0], out[1]);
      } else {
        if (jin[0]) orow[0] = out[0];
        if (jin[1]) orow[1] = out[1];
      }
    }
    __syncthreads();  // row r-1's stage is free
    if (tid == 0 && k - 1 + S < nrows) issue(k - 1 + S);
    sm = sc;
    sc = sp;
    phc = php;
    if (++sp == S) sp = 0, php ^= 1u;
  }
}

}  // namespace sgb
