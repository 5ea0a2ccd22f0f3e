// fp64 streaming gather adjoint for the 3D stars (sm_100a): the reference's
// own precision on the cfg 2 (radius 1, c or c^2, u_2 active) and cfg 4 / 5
// (radius 4, c^2) stencils.
//
// Mathematics and boundary predicate as every 3D gather kernel here (SURVEY
// Appendix C; reference adjoint.cpp:73-163 / interp.cpp:189-198):
//   u_1_b[o] += sum_l w_l q(o - o_l) + 2 u_b[o] [o in B],  q = D c^(1|2) u_b [x in B]
//   c_b[o]   += g[o] Lap(u_1)[o],      g = D u_b | 2 D c u_b  [o in B]
//   u_2_b[o] -= u_b[o] [o in B]        (radius-1 specs)
// Structure of the fp32 v7 kernel (star3d_r4.cuh) re-balanced for doubles,
// where the shared-memory pipe -- not DRAM -- bounded the plane kernel it
// replaces (star3d_plane.cuh: one point per thread, 17 shared loads per
// point and field, ncu mio_throttle / barrier stalls, profiles/):
//   * one CTA per SM (512 threads) owns a 32 (k) x 32 (j) column tile and
//     streams over i; per plane one elected thread issues TMA loads of the
//     c / u_b / u_1 halo boxes and the c_b / u_1_b tiles of the output plane
//     o = p - R (and the u_2_b tile of plane p) into a 3-stage mbarrier ring;
//   * the seed map is windowed to the primal box, so TMA's zero fill is the
//     seed mask in j and k (the i test is per plane);
//   * warps 0-7 carry Lap(u_1) (emit c_b), warps 8-15 the q stencil (emit
//     u_1_b); each thread owns 2 rows x 2 k points of one field: k neighbours
//     from a 16-byte-load window per row, j neighbours from shared rows
//     common to its two rows, i in 2R+1 rotating accumulators -- at radius 4
//     4.5 16-byte shared loads per point and field instead of 17 8-byte ones;
//   * g is formed in the q-pass; one q buffer and an R+1-slot g ring (smem
//     budget), so a second barrier per plane closes the q / g reuse.
#pragma once

#include "star3d_plane.cuh"
#include "star3d_r4.cuh"

namespace sgb {

template <int MODE>
struct StarTileD {
  static constexpr int R = Star3<MODE>::R;
  static constexpr int TK = 32, TJ = 32, HJ = R;
  static constexpr int HK = R > 2 ? R : 2;  // k halo: >= R, even (16-byte loads)
  static constexpr int BW = TK + 2 * HK;    // box row (40 / 36 doubles)
  static constexpr int BJ = TJ + 2 * HJ;
  static constexpr int RING = 2 * R + 1;
  static constexpr int NS = 3;
  static constexpr int QD = R + 1;
  static constexpr int ROLE = (TK / 2) * (TJ / 2);  // 256 threads per field
  static constexpr int THREADS = 2 * ROLE;
  static constexpr int BOX = BW * BJ;
  static constexpr int BP = (BOX + 15) / 16 * 16;  // box slot stride: 128-byte aligned
  static constexpr int TILE = TK * TJ;
  static constexpr int NT = Star3<MODE>::kU2 ? 3 : 2;  // c_b, u_1_b (, u_2_b) tiles
  static constexpr int SF = 3 * BP + NT * TILE;
  static constexpr int QPAIRS = BOX / 2;
  static constexpr int EPT = (QPAIRS + THREADS - 1) / THREADS;
  static constexpr size_t SMEM = (size_t)(NS * SF + BP + QD * TILE) * 8 + 2 * NS * 8;
  static_assert(RING % NS == 0, "static stage index");
  static_assert((TILE * 8) % 128 == 0, "TMA destinations 128-B aligned");
  static_assert(SMEM <= 227 * 1024, "shared memory");
};

__device__ __forceinline__ double2 ldd2(const double* p) {
  return *reinterpret_cast<const double2*>(p);
}
__device__ __forceinline__ double2 fmad2(double w, const double2& v, const double2& a) {
  return make_double2(fma(w, v.x, a.x), fma(w, v.y, a.y));
}

// in-plane k stencil of 2 points (k, k+1) of one row: window k-HK .. k+HK+1
template <int R, int HK>
__device__ __forceinline__ double2 kstencil_d(const double* row, double w0,
                                              const double (&wr)[R + 1]) {
  double kw[2 * HK + 2];
#pragma unroll
  for (int q = 0; q <= HK; q++) {
    const double2 v = ldd2(row - HK + 2 * q);
    kw[2 * q] = v.x;
    kw[2 * q + 1] = v.y;
  }
  double p0 = w0 * kw[HK], p1 = w0 * kw[HK + 1];
#pragma unroll
  for (int r = 1; r <= R; r++) {
    p0 = fma(wr[r], kw[HK - r] + kw[HK + r], p0);
    p1 = fma(wr[r], kw[HK + 1 - r] + kw[HK + 1 + r], p1);
  }
  return make_double2(p0, p1);
}

// 2 rows x 2 k of one field, plane phase ph: in-plane stencil into acc[ph],
// the plane's centre values into the i-neighbours' accumulators.
template <int MODE>
__device__ __forceinline__ void field2x2_d(const double* F, int r0, int col, double w0,
                                           const double (&wr)[StarTileD<MODE>::R + 1],
                                           double2 (&acc)[StarTileD<MODE>::RING][2], int ph) {
  constexpr int BW = StarTileD<MODE>::BW, HK = StarTileD<MODE>::HK;
  constexpr int R = StarTileD<MODE>::R, RING = StarTileD<MODE>::RING;
  const double* row0 = F + r0 * BW + col;
  const double2 b0 = ldd2(row0), b1 = ldd2(row0 + BW);
  double2 in0 = kstencil_d<R, HK>(row0, w0, wr);
  double2 in1 = kstencil_d<R, HK>(row0 + BW, w0, wr);
  in0 = fmad2(wr[1], b1, in0);
  in1 = fmad2(wr[1], b0, in1);
#pragma unroll
  for (int t = -R; t <= R + 1; t++) {
    if (t == 0 || t == 1) continue;
    const double2 v = ldd2(row0 + t * BW);
    const int d0 = t < 0 ? -t : t, d1 = t - 1 < 0 ? 1 - t : t - 1;
    if (d0 <= R) in0 = fmad2(wr[d0], v, in0);
    if (d1 <= R) in1 = fmad2(wr[d1], v, in1);
  }
  acc[ph][0] = make_double2(acc[ph][0].x + in0.x, acc[ph][0].y + in0.y);
  acc[ph][1] = make_double2(acc[ph][1].x + in1.x, acc[ph][1].y + in1.y);
  acc[(ph + R) % RING][0] = make_double2(wr[R] * b0.x, wr[R] * b0.y);
  acc[(ph + R) % RING][1] = make_double2(wr[R] * b1.x, wr[R] * b1.y);
#pragma unroll
  for (int r = 1; r <= R; r++) {
    if (r < R) {
      acc[(ph + r) % RING][0] = fmad2(wr[r], b0, acc[(ph + r) % RING][0]);
      acc[(ph + r) % RING][1] = fmad2(wr[r], b1, acc[(ph + r) % RING][1]);
    }
    acc[(ph + RING - r) % RING][0] = fmad2(wr[r], b0, acc[(ph + RING - r) % RING][0]);
    acc[(ph + RING - r) % RING][1] = fmad2(wr[r], b1, acc[(ph + RING - r) % RING][1]);
  }
}

// UBW: the u_b map is windowed to [lo, hi]^2 (TMA zero fill = seed mask);
// otherwise the mask is applied in the q-pass and the centre term.
template <int MODE, bool UBW>
__global__ void __launch_bounds__(StarTileD<MODE>::THREADS, 1)
    star3_f64_stream_kernel(const __grid_constant__ CUtensorMap tm_c,
                            const __grid_constant__ CUtensorMap tm_ub,
                            const __grid_constant__ CUtensorMap tm_u1,
                            const __grid_constant__ CUtensorMap tm_cb,
                            const __grid_constant__ CUtensorMap tm_u1b,
                            const __grid_constant__ CUtensorMap tm_u2b,
                            double* __restrict__ c_b, double* __restrict__ u_1_b,
                            double* __restrict__ u_2_b, int n, int i_base, int lo, int hi,
                            int out_i0, int out_i1, int chunk, int tiles_k, double D) {
  using Tl = StarTileD<MODE>;
  using S3 = Star3<MODE>;
  constexpr int R = Tl::R, HJ = Tl::HJ, HK = Tl::HK, BW = Tl::BW, TK = Tl::TK;
  constexpr int RING = Tl::RING, NS = Tl::NS, BOX = Tl::BOX, BP = Tl::BP, QD = Tl::QD;
  constexpr int SF = Tl::SF, TILE = Tl::TILE, ROLE = Tl::ROLE;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stage = reinterpret_cast<double*>(smem_raw);  // [NS][c, ub, u1 boxes | tiles]
  double* Q = stage + NS * SF;                          // q box
  double* gq = Q + BP;                                  // [QD][TJ][TK] g of centres
  uint64_t* bars = reinterpret_cast<uint64_t*>(gq + QD * TILE);

  const int tid = threadIdx.x;
  const bool q_role = tid >= ROLE;  // warp-uniform
  const int rt = q_role ? tid - ROLE : tid;
  const int tx = rt & 15, ty = rt >> 4;  // 2 k-points x rows 2ty, 2ty+1
  const int tk = blockIdx.x % tiles_k, tj = blockIdx.x / tiles_k;
  const int k0 = tk * TK, j0 = tj * Tl::TJ;
  const int o_begin = out_i0 + blockIdx.y * chunk;
  const int o_end = min(o_begin + chunk, out_i1);
  if (o_begin >= o_end) return;
  const int pstart = o_begin - R;
  const int P = (o_end - o_begin) + 2 * R;

  const double w0 = S3::template w<double>(0);
  double wr[R + 1];
  wr[0] = w0;
#pragma unroll
  for (int r = 1; r <= R; r++) wr[r] = S3::template w<double>(r);

  // Fresh form (MODE 4): split stage barriers as in the fp32 v8 kernel -- the
  // c / u_b boxes (A half; read only by the q pass, before the plane's first
  // barrier) complete on their own mbarrier and are requested a plane earlier
  // than the u_1 box and the c_b tile (B half).  The accumulating forms keep
  // one barrier per stage (the split loses there, as it does in fp32).
  constexpr bool SPLIT = S3::kU1bFresh && !S3::kU2;
  uint64_t* barsB = bars + NS;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < (SPLIT ? 2 * NS : NS); s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  __syncthreads();
  auto issueA = [&](int it) {  // c, u_b boxes (the whole stage when !SPLIT)
    const int s = it % NS;
    double* dst = stage + s * SF;
    const int pl = pstart + it - i_base;
    const bool emit = it >= 2 * R;
    const int p = pstart + it;
    const bool u2 = S3::kU2 && p >= o_begin && p < o_end;  // u_2_b tile of plane p
    // fresh u_1_b (MODE 4): its old tile is not needed
    tma::mbar_arrive_expect_tx(
        &bars[s],
        SPLIT ? 2 * BOX * 8
              : (3 * BOX + ((emit ? (S3::kU1bFresh ? 1 : 2) : 0) + (u2 ? 1 : 0)) * TILE) * 8);
    tma::load_3d(dst, &tm_c, &bars[s], k0 - HK, j0 - HJ, pl);
    tma::load_3d(dst + BP, &tm_ub, &bars[s], k0 - HK - (UBW ? lo : 0), j0 - HJ - (UBW ? lo : 0),
                 pl);
    if (SPLIT) return;
    tma::load_3d(dst + 2 * BP, &tm_u1, &bars[s], k0 - HK, j0 - HJ, pl);
    if (emit) {
      tma::load_3d(dst + 3 * BP, &tm_cb, &bars[s], k0, j0, pl - R);
      if (!S3::kU1bFresh) tma::load_3d(dst + 3 * BP + TILE, &tm_u1b, &bars[s], k0, j0, pl - R);
    }
    if (u2) tma::load_3d(dst + 3 * BP + 2 * TILE, &tm_u2b, &bars[s], k0, j0, pl);
  };
  auto issueB = [&](int it) {  // SPLIT only: u_1 box and the c_b tile of the output plane
    const int s = it % NS;
    double* dst = stage + s * SF;
    const int pl = pstart + it - i_base;
    const bool emit = it >= 2 * R;
    tma::mbar_arrive_expect_tx(&barsB[s], (BOX + (emit ? TILE : 0)) * 8);
    tma::load_3d(dst + 2 * BP, &tm_u1, &barsB[s], k0 - HK, j0 - HJ, pl);
    if (emit) tma::load_3d(dst + 3 * BP, &tm_cb, &barsB[s], k0, j0, pl - R);
  };
  if (tid == 0)
    for (int it = 0; it < NS && it < P; it++) {
      issueA(it);
      if (SPLIT) issueB(it);
    }

  const int jr0 = j0 + 2 * ty, kc = k0 + 2 * tx;
  const int r0 = 2 * ty + HJ, col = HK + 2 * tx;
  const int trow = 2 * ty * TK + 2 * tx;  // row 2ty of a 32x32 tile
  const long long plane = (long long)n * n;
  const long long coff = (long long)jr0 * n + kc;

  // q-pass pairs of this thread: box offset and, for centres, g-tile offset
  int qoff[Tl::EPT], goff[Tl::EPT];
  uint32_t qmask = 0;  // !UBW: bit 2m+x = element x of pair m inside [lo, hi]^2
#pragma unroll
  for (int m = 0; m < Tl::EPT; m++) {
    const int e = tid + m * Tl::THREADS;
    const int row = e / (BW / 2), c2 = e - row * (BW / 2);
    qoff[m] = e < Tl::QPAIRS ? row * BW + 2 * c2 : -1;
    const int jg = j0 - HJ + row, kg = k0 - HK + 2 * c2;
#pragma unroll
    for (int x = 0; x < 2; x++)
      if (jg >= lo && jg <= hi && kg + x >= lo && kg + x <= hi) qmask |= 1u << (2 * m + x);
    goff[m] = (e < Tl::QPAIRS && row >= HJ && row < HJ + Tl::TJ && c2 >= HK / 2 &&
               c2 < HK / 2 + TK / 2)
                  ? (row - HJ) * TK + 2 * (c2 - HK / 2)
                  : -1;
  }
  // per-point masks (plane-independent): bit 2h+x for point (jr0+h, kc+x)
  //   inb : j, k in [lo, hi];  one : exactly one of j, k outside, by <= R
  //   grid (bits 4, 5): row h inside the grid (kc < n, n even: kc+1 < n too)
  uint32_t inb = 0, one = 0, grid = 0;
#pragma unroll
  for (int h = 0; h < 2; h++) {
    const int j = jr0 + h;
    if (j < n && kc < n) grid |= 1u << h;
    const int jout = j < lo ? lo - j : (j > hi ? j - hi : 0);
#pragma unroll
    for (int x = 0; x < 2; x++) {
      const int k = kc + x;
      const int kout = k < lo ? lo - k : (k > hi ? k - hi : 0);
      if (jout == 0 && kout == 0) inb |= 1u << (2 * h + x);
      if ((jout > 0) + (kout > 0) == 1 && jout <= R && kout <= R) one |= 1u << (2 * h + x);
    }
  }

  double2 acc[RING][2];
#pragma unroll
  for (int s = 0; s < RING; s++) acc[s][0] = acc[s][1] = make_double2(0.0, 0.0);

  for (int base = 0; base < P; base += RING) {
    const int par0 = base / NS;
#pragma unroll
    for (int ph = 0; ph < RING; ph++) {
      const int it = base + ph;
      if (it < P) {
        const int s = ph % NS;
        const int p = pstart + it;
        const double* Cs = stage + s * SF;
        const double* UBs = Cs + BP;
        const double* U1s = Cs + 2 * BP;
        double* G = gq + (it % QD) * TILE;
        const int o = p - R;
        const bool pin = p >= lo && p <= hi;

        tma::mbar_wait(&bars[s], (par0 + ph / NS) & 1);
        // ---- q over the halo box; g for the centre pairs
#pragma unroll
        for (int m = 0; m < Tl::EPT; m++) {
          if (qoff[m] >= 0) {
            const int qo = qoff[m];
            double2 qv = make_double2(0.0, 0.0), gv = qv;
            if (pin) {
              const double2 cv = ldd2(Cs + qo);
              double2 uv = ldd2(UBs + qo);
              if (!UBW)
                uv = make_double2((qmask >> (2 * m)) & 1 ? uv.x : 0.0,
                                  (qmask >> (2 * m + 1)) & 1 ? uv.y : 0.0);
              const double2 du = make_double2(D * uv.x, D * uv.y);
              if (S3::kC2) {  // q = D c^2 u_b, g = 2 D c u_b
                qv = make_double2(cv.x * cv.x * du.x, cv.y * cv.y * du.y);
                gv = make_double2(2.0 * cv.x * du.x, 2.0 * cv.y * du.y);
              } else {        // q = D c u_b, g = D u_b
                qv = make_double2(cv.x * du.x, cv.y * du.y);
                gv = du;
              }
            }
            *reinterpret_cast<double2*>(Q + qo) = qv;
            if (goff[m] >= 0) *reinterpret_cast<double2*>(G + goff[m]) = gv;
          }
        }
        // ---- q role: the 2 u_b centre term of output plane p, and the u_2
        // partial u_2_b[p] -= u_b[p] on B (radius-1 specs) at plane p itself
        if (q_role && pin) {
#pragma unroll
          for (int h = 0; h < 2; h++) {
            double2 ubm = ldd2(UBs + (r0 + h) * BW + col);
            if (!UBW)
              ubm = make_double2((inb >> (2 * h)) & 1 ? ubm.x : 0.0,
                                 (inb >> (2 * h + 1)) & 1 ? ubm.y : 0.0);
            acc[ph][h] = fmad2(2.0, ubm, acc[ph][h]);
            if (S3::kU2 && p >= o_begin && p < o_end) {
              const uint32_t mk = inb >> (2 * h);
              if (((grid >> h) & 1) && (mk & 3)) {
                const double2 u2 = ldd2(Cs + 3 * BP + 2 * TILE + trow + h * TK);
                const double2 nv = make_double2((mk & 1) ? u2.x + -ubm.x : u2.x,
                                                (mk & 2) ? u2.y + -ubm.y : u2.y);
                __stcs(reinterpret_cast<double2*>(u_2_b + (long long)(p - i_base) * plane +
                                                  coff + h * n),
                       nv);
              }
            }
          }
        }
        __syncthreads();  // Q / G of plane p complete; stage of plane p-1 free
        if (tid == 0) {
          if (SPLIT) {  // B of plane it-1+NS first (needed first), then A of plane it+NS
            if (it >= 1 && it - 1 + NS < P) issueB(it - 1 + NS);
            if (it + NS < P) issueA(it + NS);
          } else if (it >= 1 && it - 1 + NS < P) {
            issueA(it - 1 + NS);
          }
        }
        if (SPLIT) tma::mbar_wait(&barsB[s], (par0 + ph / NS) & 1);

        field2x2_d<MODE>(q_role ? Q : U1s, r0, col, w0, wr, acc, ph);

        // ---- emit output plane o = p - R
        if (it >= 2 * R) {
          const int es = (ph + R + 1) % RING;
          const long long obase = (long long)(o - i_base) * plane;
          const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
          const double* OLD = Cs + 3 * BP + (q_role ? TILE : 0) + trow;
          if (!q_role) {
            if (oout == 0) {
              const double* Go = gq + ((it - R) % QD) * TILE + trow;
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const uint32_t mk = inb >> (2 * h);
                if (!((grid >> h) & 1) || !(mk & 3)) continue;
                const double2 old = ldd2(OLD + h * TK), g = ldd2(Go + h * TK);
                const double2 a = acc[es][h];
                const double2 nv = make_double2((mk & 1) ? fma(g.x, a.x, old.x) : old.x,
                                                (mk & 2) ? fma(g.y, a.y, old.y) : old.y);
                __stcs(reinterpret_cast<double2*>(c_b + obase + coff + h * n), nv);
              }
            }
          } else {
            // reached iff at most one coordinate is outside [lo, hi], by <= R;
            // MODE 4 writes every grid point (0 + sum where reached, else 0)
            const uint32_t reach = oout == 0 ? (inb | one) : (oout <= R ? inb : 0u);
#pragma unroll
            for (int h = 0; h < 2; h++) {
              const uint32_t mk = reach >> (2 * h);
              if (!((grid >> h) & 1) || (!S3::kU1bFresh && !(mk & 3))) continue;
              const double2 old =
                  S3::kU1bFresh ? make_double2(0.0, 0.0) : ldd2(OLD + h * TK);
              const double2 a = acc[es][h];
              const double2 nv = make_double2((mk & 1) ? old.x + a.x : old.x,
                                              (mk & 2) ? old.y + a.y : old.y);
              __stcs(reinterpret_cast<double2*>(u_1_b + obase + coff + h * n), nv);
            }
          }
        }
        __syncthreads();  // Q and the emitted g slot free for the next plane
      }
    }
  }
}

// v8 form of the fp64 radius-4 gather (MODE 2 / 4, windowed seed map; opt-in,
// SGB_F64_V8=1 -- measured no faster, see the launcher): 256
// threads, each 4 rows x 2 k of one field -- the j rows shared by a thread's
// 4 rows halve the shared-memory row loads per point (the kernel above is
// bound by the shared-memory pipe) -- every term in field2x2_d's order
// (bitwise equal to star3_f64_stream_kernel), and split stage barriers: the
// c / u_b boxes (read only by the q pass) are requested right after the
// plane's first barrier, a plane before the u_1 box and output tiles.
template <int MODE>
struct StarTileD8 : StarTileD<MODE> {
  static constexpr int ROLE = (StarTileD<MODE>::TK / 2) * (StarTileD<MODE>::TJ / 4);  // 128
  static constexpr int THREADS = 2 * ROLE;
  static constexpr int EPT = (StarTileD<MODE>::QPAIRS + THREADS - 1) / THREADS;
  static constexpr size_t SMEM = StarTileD<MODE>::SMEM + StarTileD<MODE>::NS * 8;
};

template <int MODE>
__device__ __forceinline__ void field4x2_d(const double* F, int r0, int col, double w0,
                                           const double (&wr)[StarTileD<MODE>::R + 1],
                                           double2 (&acc)[StarTileD<MODE>::RING][4], int ph) {
  constexpr int BW = StarTileD<MODE>::BW, HK = StarTileD<MODE>::HK;
  constexpr int R = StarTileD<MODE>::R, RING = StarTileD<MODE>::RING;
  const double* row0 = F + r0 * BW + col;
  double2 b[4], in[4];
#pragma unroll
  for (int h = 0; h < 4; h++) {
    b[h] = ldd2(row0 + h * BW);
    in[h] = kstencil_d<R, HK>(row0 + h * BW, w0, wr);
  }
  // field2x2_d's per-row order: the pair partner, then the rows bottom to top
#pragma unroll
  for (int pos = 0; pos < 2 * R; pos++) {
#pragma unroll
    for (int h = 0; h < 4; h++) {
      int off;
      if ((h & 1) == 0) off = pos == 0 ? 1 : (pos <= R ? pos - 1 - R : pos - R + 1);
      else off = pos == 0 ? -1 : (pos < R ? pos - 1 - R : pos - R + 1);
      const int t = h + off;
      const int d = off < 0 ? -off : off;
      const double2 v =
          (t >= 0 && t <= 3) ? b[t < 0 ? 0 : (t > 3 ? 3 : t)] : ldd2(row0 + t * BW);
      in[h] = fmad2(wr[d], v, in[h]);
    }
  }
#pragma unroll
  for (int h = 0; h < 4; h++) {
    acc[ph][h] = make_double2(acc[ph][h].x + in[h].x, acc[ph][h].y + in[h].y);
    acc[(ph + R) % RING][h] = make_double2(wr[R] * b[h].x, wr[R] * b[h].y);
#pragma unroll
    for (int r = 1; r <= R; r++) {
      if (r < R) acc[(ph + r) % RING][h] = fmad2(wr[r], b[h], acc[(ph + r) % RING][h]);
      acc[(ph + RING - r) % RING][h] = fmad2(wr[r], b[h], acc[(ph + RING - r) % RING][h]);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(StarTileD8<MODE>::THREADS, 1)
    star3_f64_v8_kernel(const __grid_constant__ CUtensorMap tm_c,
                        const __grid_constant__ CUtensorMap tm_ub,
                        const __grid_constant__ CUtensorMap tm_u1,
                        const __grid_constant__ CUtensorMap tm_cb,
                        const __grid_constant__ CUtensorMap tm_u1b, double* __restrict__ c_b,
                        double* __restrict__ u_1_b, int n, int i_base, int lo, int hi,
                        int out_i0, int out_i1, int chunk, int tiles_k, double D) {
  using Tl = StarTileD8<MODE>;
  using S3 = Star3<MODE>;
  static_assert(!S3::kU2 && !S3::kU2Set, "fp64 v8: radius-4 specs without u_2 partials");
  constexpr int R = Tl::R, HJ = Tl::HJ, HK = Tl::HK, BW = Tl::BW, TK = Tl::TK;
  constexpr int RING = Tl::RING, NS = Tl::NS, BOX = Tl::BOX, BP = Tl::BP, QD = Tl::QD;
  constexpr int SF = Tl::SF, TILE = Tl::TILE, ROLE = Tl::ROLE;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stage = reinterpret_cast<double*>(smem_raw);
  double* Q = stage + NS * SF;
  double* gq = Q + BP;
  uint64_t* bars = reinterpret_cast<uint64_t*>(gq + QD * TILE);
  uint64_t* barsB = bars + NS;

  const int tid = threadIdx.x;
  const bool q_role = tid >= ROLE;
  const int rt = q_role ? tid - ROLE : tid;
  const int tx = rt & 15, ty = rt >> 4;  // 2 k-points x rows 4ty .. 4ty+3
  const int tk = blockIdx.x % tiles_k, tj = blockIdx.x / tiles_k;
  const int k0 = tk * TK, j0 = tj * Tl::TJ;
  const int o_begin = out_i0 + blockIdx.y * chunk;
  const int o_end = min(o_begin + chunk, out_i1);
  if (o_begin >= o_end) return;
  const int pstart = o_begin - R;
  const int P = (o_end - o_begin) + 2 * R;

  const double w0 = S3::template w<double>(0);
  double wr[R + 1];
  wr[0] = w0;
#pragma unroll
  for (int r = 1; r <= R; r++) wr[r] = S3::template w<double>(r);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < 2 * NS; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  __syncthreads();
  auto issueA = [&](int it) {
    const int s = it % NS;
    double* dst = stage + s * SF;
    const int pl = pstart + it - i_base;
    tma::mbar_arrive_expect_tx(&bars[s], 2 * BOX * 8);
    tma::load_3d(dst, &tm_c, &bars[s], k0 - HK, j0 - HJ, pl);
    tma::load_3d(dst + BP, &tm_ub, &bars[s], k0 - HK - lo, j0 - HJ - lo, pl);
  };
  auto issueB = [&](int it) {
    const int s = it % NS;
    double* dst = stage + s * SF;
    const int pl = pstart + it - i_base;
    const bool emit = it >= 2 * R;
    tma::mbar_arrive_expect_tx(&barsB[s],
                               (BOX + (emit ? (S3::kU1bFresh ? 1 : 2) : 0) * TILE) * 8);
    tma::load_3d(dst + 2 * BP, &tm_u1, &barsB[s], k0 - HK, j0 - HJ, pl);
    if (emit) {
      tma::load_3d(dst + 3 * BP, &tm_cb, &barsB[s], k0, j0, pl - R);
      if (!S3::kU1bFresh) tma::load_3d(dst + 3 * BP + TILE, &tm_u1b, &barsB[s], k0, j0, pl - R);
    }
  };
  if (tid == 0)
    for (int it = 0; it < NS && it < P; it++) {
      issueA(it);
      issueB(it);
    }

  const int jr0 = j0 + 4 * ty, kc = k0 + 2 * tx;
  const int r0 = 4 * ty + HJ, col = HK + 2 * tx;
  const int trow = 4 * ty * TK + 2 * tx;
  const long long plane = (long long)n * n;
  const long long coff = (long long)jr0 * n + kc;

  int qoff[Tl::EPT], goff[Tl::EPT];
#pragma unroll
  for (int m = 0; m < Tl::EPT; m++) {
    const int e = tid + m * Tl::THREADS;
    const int row = e / (BW / 2), c2 = e - row * (BW / 2);
    qoff[m] = e < Tl::QPAIRS ? row * BW + 2 * c2 : -1;
    goff[m] = (e < Tl::QPAIRS && row >= HJ && row < HJ + Tl::TJ && c2 >= HK / 2 &&
               c2 < HK / 2 + TK / 2)
                  ? (row - HJ) * TK + 2 * (c2 - HK / 2)
                  : -1;
  }
  // per-point masks: bit 2h+x for point (jr0+h, kc+x); grid bit h: row inside
  uint32_t inb = 0, one = 0, grid = 0;
#pragma unroll
  for (int h = 0; h < 4; h++) {
    const int j = jr0 + h;
    if (j < n && kc < n) grid |= 1u << h;
    const int jout = j < lo ? lo - j : (j > hi ? j - hi : 0);
#pragma unroll
    for (int x = 0; x < 2; x++) {
      const int k = kc + x;
      const int kout = k < lo ? lo - k : (k > hi ? k - hi : 0);
      if (jout == 0 && kout == 0) inb |= 1u << (2 * h + x);
      if ((jout > 0) + (kout > 0) == 1 && jout <= R && kout <= R) one |= 1u << (2 * h + x);
    }
  }

  double2 acc[RING][4];
#pragma unroll
  for (int s = 0; s < RING; s++)
#pragma unroll
    for (int h = 0; h < 4; h++) acc[s][h] = make_double2(0.0, 0.0);

  for (int base = 0; base < P; base += RING) {
    const int par0 = base / NS;
#pragma unroll
    for (int ph = 0; ph < RING; ph++) {
      const int it = base + ph;
      if (it < P) {
        const int s = ph % NS;
        const int p = pstart + it;
        const double* Cs = stage + s * SF;
        const double* UBs = Cs + BP;
        const double* U1s = Cs + 2 * BP;
        double* G = gq + (it % QD) * TILE;
        const int o = p - R;
        const bool pin = p >= lo && p <= hi;
        const uint32_t par = (par0 + ph / NS) & 1;

        tma::mbar_wait(&bars[s], par);
#pragma unroll
        for (int m = 0; m < Tl::EPT; m++) {
          if (qoff[m] >= 0) {
            const int qo = qoff[m];
            double2 qv = make_double2(0.0, 0.0), gv = qv;
            if (pin) {
              const double2 cv = ldd2(Cs + qo);
              const double2 uv = ldd2(UBs + qo);
              const double2 du = make_double2(D * uv.x, D * uv.y);
              qv = make_double2(cv.x * cv.x * du.x, cv.y * cv.y * du.y);
              gv = make_double2(2.0 * cv.x * du.x, 2.0 * cv.y * du.y);
            }
            *reinterpret_cast<double2*>(Q + qo) = qv;
            if (goff[m] >= 0) *reinterpret_cast<double2*>(G + goff[m]) = gv;
          }
        }
        if (q_role && pin) {
#pragma unroll
          for (int h = 0; h < 4; h++)
            acc[ph][h] = fmad2(2.0, ldd2(UBs + (r0 + h) * BW + col), acc[ph][h]);
        }
        __syncthreads();  // Q / G of plane p complete; A half of stage s and the
                          // B half of plane p-1's stage free
        if (tid == 0) {
          if (it + NS < P) issueA(it + NS);
          if (it >= 1 && it - 1 + NS < P) issueB(it - 1 + NS);
        }
        tma::mbar_wait(&barsB[s], par);

        field4x2_d<MODE>(q_role ? Q : U1s, r0, col, w0, wr, acc, ph);

        if (it >= 2 * R) {
          const int es = (ph + R + 1) % RING;
          const long long obase = (long long)(o - i_base) * plane;
          const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
          const double* OLD = Cs + 3 * BP + (q_role ? TILE : 0) + trow;
          if (!q_role) {
            if (oout == 0) {
              const double* Go = gq + ((it - R) % QD) * TILE + trow;
#pragma unroll
              for (int h = 0; h < 4; h++) {
                const uint32_t mk = inb >> (2 * h);
                if (!((grid >> h) & 1) || !(mk & 3)) continue;
                const double2 old = ldd2(OLD + h * TK), g = ldd2(Go + h * TK);
                const double2 a = acc[es][h];
                const double2 nv = make_double2((mk & 1) ? fma(g.x, a.x, old.x) : old.x,
                                                (mk & 2) ? fma(g.y, a.y, old.y) : old.y);
                __stcs(reinterpret_cast<double2*>(c_b + obase + coff + h * n), nv);
              }
            }
          } else {
            const uint32_t reach = oout == 0 ? (inb | one) : (oout <= R ? inb : 0u);
#pragma unroll
            for (int h = 0; h < 4; h++) {
              const uint32_t mk = reach >> (2 * h);
              if (!((grid >> h) & 1) || (!S3::kU1bFresh && !(mk & 3))) continue;
              const double2 old =
                  S3::kU1bFresh ? make_double2(0.0, 0.0) : ldd2(OLD + h * TK);
              const double2 a = acc[es][h];
              const double2 nv = make_double2((mk & 1) ? old.x + a.x : old.x,
                                              (mk & 2) ? old.y + a.y : old.y);
              __stcs(reinterpret_cast<double2*>(u_1_b + obase + coff + h * n), nv);
            }
          }
        }
        __syncthreads();  // Q and the emitted g slot free for the next plane
      }
    }
  }
}

// Same-shape TMA map restricted to the window [off, off+ext) in j and k
// (TMA zero fill outside = the seed mask); needs a 16-byte aligned window base.
inline int encode_3d_window_f64(CUtensorMap* map, const double* base, long long n,
                                long long nplanes, long long off, long long ext, int box0,
                                int box1, const char* name) {
  const double* wb = base + off * n + off;
  if ((reinterpret_cast<uintptr_t>(wb) & 15) != 0 || ext < 1) return 1;
  auto encode = get_encode();
  if (!encode) {
    set_error(std::string(name) + ": cuTensorMapEncodeTiled unavailable");
    return SGB_EINVAL;
  }
  cuuint64_t dims[3] = {(cuuint64_t)ext, (cuuint64_t)ext, (cuuint64_t)nplanes};
  cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)n * n * 8};
  cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)wb, dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(std::string(name) + ": tensor map encode failed (" + std::to_string((int)r) + ")");
    return SGB_EINVAL;
  }
  return 0;
}

// Host launcher; returns 1 when the shape does not fit this kernel (the
// caller uses the plane / per-point kernels), 0 / negative like the others.
template <int MODE>
inline int star3_f64_stream_gather(const Slab3& g, long long lo, long long hi, long long out_i0,
                                   long long out_i1, double D, const double* c, double* c_b,
                                   const double* u_1, double* u_1_b, double* u_2_b,
                                   const double* u_b, cudaStream_t s, const char* name) {
  using Tl = StarTileD<MODE>;
  constexpr bool kU2 = Star3<MODE>::kU2;
  if (g.n % 2 != 0 || g.n > (1 << 20) || g.n < 2 * Tl::R + 2 || hi < lo) return 1;
  for (const void* p : {(const void*)c, (const void*)c_b, (const void*)u_1, (const void*)u_1_b,
                        (const void*)u_b, (const void*)(kU2 ? u_2_b : u_1_b)})
    if (reinterpret_cast<uintptr_t>(p) & 15) return 1;
  CUtensorMap maps[6];
  int rc = encode_3d_t(&maps[0], c, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  const int w = encode_3d_window_f64(&maps[1], u_b, g.n, g.nplanes, lo, hi - lo + 1, Tl::BW,
                                     Tl::BJ, name);
  if (w < 0) return w;
  const bool ubw = w == 0;  // else (odd lo*(n+1)): full map, mask in the kernel
  if (!ubw) rc |= encode_3d_t(&maps[1], u_b, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  rc |= encode_3d_t(&maps[2], u_1, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  rc |= encode_3d_t(&maps[3], (const double*)c_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  rc |= encode_3d_t(&maps[4], (const double*)u_1_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  rc |= encode_3d_t(&maps[5], (const double*)(kU2 ? u_2_b : u_1_b), g.n, g.nplanes, Tl::TK,
                    Tl::TJ, name);
  if (rc) return SGB_EINVAL;
  if (int rc = ensure_smem((const void*)star3_f64_stream_kernel<MODE, true>, Tl::SMEM, name))
    return rc;
  if (int rc = ensure_smem((const void*)star3_f64_stream_kernel<MODE, false>, Tl::SMEM, name))
    return rc;
  const int tiles_k = (int)((g.n + Tl::TK - 1) / Tl::TK);
  const long long tiles = (long long)tiles_k * ((g.n + Tl::TJ - 1) / Tl::TJ);
  const long long nout = out_i1 - out_i0;
  // i-chunks: the wave model of star3d_r4.cuh (one CTA per SM, equal-length CTAs)
  int nch = 0;
  if (opt(OPT_F64_ICHUNKS, 0) > 0) nch = (int)opt(OPT_F64_ICHUNKS, 0);
  if (nch == 0) {
    const int sms = num_sms();
    long long best = -1;
    for (int cc = 1; cc <= 64 && cc <= nout; cc++) {
      const long long len = (nout + cc - 1) / cc;
      const long long waves = (tiles * cc + sms - 1) / sms;
      const long long cost = waves * (len + 2 * Tl::R);
      if (best < 0 || cost < best) best = cost, nch = cc;
    }
  }
  const int chunk = (int)((nout + nch - 1) / nch);
  const unsigned gy = (unsigned)((nout + chunk - 1) / chunk);
  if constexpr (MODE == 2 || MODE == 4) {
    // the v8 form (bitwise the same result): not faster here -- 768^3 4.48
    // vs 4.52 ms accumulating, 4.27 vs 4.43 ms fresh; 1024^3 10.75 vs 10.70
    // / 10.08 vs 10.31 ms (scripts/f64v8_check.py) -- so it is opt-in
    if (ubw && opt(OPT_F64_V8, 0)) {
      using T8 = StarTileD8<MODE>;
      if (int rc = ensure_smem((const void*)star3_f64_v8_kernel<MODE>, T8::SMEM, name)) return rc;
      star3_f64_v8_kernel<MODE><<<dim3((unsigned)tiles, gy), T8::THREADS, T8::SMEM, s>>>(
          maps[0], maps[1], maps[2], maps[3], maps[4], c_b, u_1_b, (int)g.n, (int)g.i_base,
          (int)lo, (int)hi, (int)out_i0, (int)out_i1, chunk, tiles_k, D);
      return launch_status(name);
    }
  }
  auto kern = ubw ? star3_f64_stream_kernel<MODE, true> : star3_f64_stream_kernel<MODE, false>;
  kern<<<dim3((unsigned)tiles, gy), Tl::THREADS, Tl::SMEM, s>>>(
      maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], c_b, u_1_b, u_2_b, (int)g.n,
      (int)g.i_base, (int)lo, (int)hi, (int)out_i0, (int)out_i1, chunk, tiles_k, D);
  return launch_status(name);
}

// ---------------------------------------------------------------------------
// fp64 streaming primal (run_nest semantics, interp.cpp:153-173; emitted form
// codegen.cpp:311-330): u = 2 u_1 - u_2 + c^(1|2) D Lap(u_1) on B (or += for
// the '+=' specs), points outside B untouched.  The fp32 streaming primal's
// scheme (star3d_primal.cuh) with the fp64 gather's 2 x 2 register blocking:
// 32x32 column tiles, 256 threads, per plane p the u_1 halo box and the c /
// u_2 / u_1 (/ u) tiles of the output plane o = p - R through a 3-stage TMA
// ring, ~110 KB: two CTAs per SM; ~48-plane i-chunks (the lock-step that
// made the fp32 primal reach the copy bandwidth).
template <int MODE>
struct PrimalTileD {
  static constexpr int R = Star3<MODE>::R;
  static constexpr int TK = StarTileD<MODE>::TK, TJ = StarTileD<MODE>::TJ;
  static constexpr int HK = StarTileD<MODE>::HK, HJ = R;
  static constexpr int BW = StarTileD<MODE>::BW, BJ = StarTileD<MODE>::BJ;
  static constexpr int RING = 2 * R + 1, NS = 3;
  static constexpr int THREADS = (TK / 2) * (TJ / 2);
  static constexpr int BOX = BW * BJ, BP = StarTileD<MODE>::BP, TILE = TK * TJ;
  static constexpr int NT = Star3<MODE>::kIncrement ? 4 : 3;  // c, u_2, u_1 (, u)
  static constexpr int SF = BP + NT * TILE;
  static constexpr int SMEM = NS * SF * 8 + NS * 8;
  static_assert(RING % NS == 0, "static stage index");
};

template <int MODE>
__global__ void __launch_bounds__(PrimalTileD<MODE>::THREADS, 2)
    star3_primal_f64_kernel(const __grid_constant__ CUtensorMap tm_box,
                            const __grid_constant__ CUtensorMap tm_c,
                            const __grid_constant__ CUtensorMap tm_u2,
                            const __grid_constant__ CUtensorMap tm_u1,
                            const __grid_constant__ CUtensorMap tm_u, double* __restrict__ u,
                            int n, int lo, int hi, int chunk, int tiles_k, double D) {
  using Tl = PrimalTileD<MODE>;
  using S3 = Star3<MODE>;
  constexpr int R = Tl::R, HJ = Tl::HJ, HK = Tl::HK, TK = Tl::TK, RING = Tl::RING;
  constexpr int NS = Tl::NS, BOX = Tl::BOX, BP = Tl::BP, TILE = Tl::TILE, SF = Tl::SF;
  constexpr int NT = Tl::NT;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stage = reinterpret_cast<double*>(smem_raw);  // [NS][box | c | u_2 | u_1 (| u)]
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage + NS * SF);

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int tk = blockIdx.x % tiles_k, tj = blockIdx.x / tiles_k;
  const int k0 = tk * TK, j0 = tj * Tl::TJ;
  const int o_begin = lo + blockIdx.y * chunk;
  const int o_end = min(o_begin + chunk, hi + 1);
  if (o_begin >= o_end) return;
  const int pstart = o_begin - R;
  const int P = (o_end - o_begin) + 2 * R;

  const double w0 = S3::template w<double>(0);
  double wr[R + 1];
  wr[0] = w0;
#pragma unroll
  for (int r = 1; r <= R; r++) wr[r] = S3::template w<double>(r);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int it) {
    const int s = it % NS;
    double* dst = stage + s * SF;
    const int p = pstart + it;
    const bool emit = it >= 2 * R;
    tma::mbar_arrive_expect_tx(&bars[s], (BOX + (emit ? NT * TILE : 0)) * 8);
    tma::load_3d(dst, &tm_box, &bars[s], k0 - HK, j0 - HJ, p);
    if (emit) {
      const int o = p - R;
      tma::load_3d(dst + BP, &tm_c, &bars[s], k0, j0, o);
      tma::load_3d(dst + BP + TILE, &tm_u2, &bars[s], k0, j0, o);
      tma::load_3d(dst + BP + 2 * TILE, &tm_u1, &bars[s], k0, j0, o);
      if (NT == 4) tma::load_3d(dst + BP + 3 * TILE, &tm_u, &bars[s], k0, j0, o);
    }
  };
  if (tid == 0)
    for (int it = 0; it < NS && it < P; it++) issue(it);

  const int jr0 = j0 + 2 * ty, kc = k0 + 2 * tx;
  const int r0 = 2 * ty + HJ, col = HK + 2 * tx;
  const int trow = 2 * ty * TK + 2 * tx;
  const long long plane = (long long)n * n;
  const long long coff = (long long)jr0 * n + kc;
  bool jin[2], kin[2];
#pragma unroll
  for (int h = 0; h < 2; h++) jin[h] = jr0 + h >= lo && jr0 + h <= hi;
#pragma unroll
  for (int x = 0; x < 2; x++) kin[x] = kc + x >= lo && kc + x <= hi;

  double2 acc[RING][2];
#pragma unroll
  for (int s = 0; s < RING; s++) acc[s][0] = acc[s][1] = make_double2(0.0, 0.0);

  for (int base = 0; base < P; base += RING) {
    const int par0 = base / NS;
#pragma unroll
    for (int ph = 0; ph < RING; ph++) {
      const int it = base + ph;
      if (it < P) {
        const int s = ph % NS;
        const double* F = stage + s * SF;
        tma::mbar_wait(&bars[s], (par0 + ph / NS) & 1);
        field2x2_d<MODE>(F, r0, col, w0, wr, acc, ph);
        if (it >= 2 * R) {
          const int es = (ph + R + 1) % RING;
          const int o = pstart + it - R;
          double* urow = u + (long long)o * plane + coff;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            if (!jin[h] || !(kin[0] || kin[1])) continue;
            const double* T0 = F + BP + trow + h * TK;
            const double2 cv = ldd2(T0), u2 = ldd2(T0 + TILE), u1 = ldd2(T0 + 2 * TILE);
            const double cc[2] = {S3::kC2 ? cv.x * cv.x : cv.x, S3::kC2 ? cv.y * cv.y : cv.y};
            const double a[2] = {acc[es][h].x, acc[es][h].y};
            const double v1[2] = {u1.x, u1.y}, v2[2] = {u2.x, u2.y};
            double v[2];
#pragma unroll
            for (int x = 0; x < 2; x++) v[x] = (2.0 * v1[x] - v2[x]) + (D * cc[x]) * a[x];
            if (NT == 4) {
              const double2 uo = ldd2(T0 + 3 * TILE);
              v[0] = uo.x + v[0];
              v[1] = uo.y + v[1];
            }
            if (kin[0] && kin[1]) {
              *reinterpret_cast<double2*>(urow + h * n) = make_double2(v[0], v[1]);
            } else {
#pragma unroll
              for (int x = 0; x < 2; x++)
                if (kin[x]) urow[h * n + x] = v[x];
            }
          }
        }
        __syncthreads();  // stage s consumed by every thread
        if (tid == 0 && it + NS < P) issue(it + NS);
      }
    }
  }
}

// Host launcher; returns 1 when the shape does not fit (caller uses the
// per-point kernel), 0 / negative like the other entries.
template <int MODE>
inline int star3_primal_f64_stream(long long n, double D, const double* c, const double* u_1,
                                   const double* u_2, double* u, cudaStream_t s,
                                   const char* name) {
  using Tl = PrimalTileD<MODE>;
  constexpr int R = Tl::R;
  const long long lo = R, hi = n - 1 - R;
  if (n % 2 != 0 || n < 2 * R + 2 || n > (1 << 20)) return 1;
  for (const void* p : {(const void*)c, (const void*)u_1, (const void*)u_2, (const void*)u})
    if (reinterpret_cast<uintptr_t>(p) & 15) return 1;
  CUtensorMap maps[5];
  int rc = 0;
  rc |= encode_3d_t(&maps[0], u_1, n, n, Tl::BW, Tl::BJ, name);
  rc |= encode_3d_t(&maps[1], c, n, n, Tl::TK, Tl::TJ, name);
  rc |= encode_3d_t(&maps[2], u_2, n, n, Tl::TK, Tl::TJ, name);
  rc |= encode_3d_t(&maps[3], u_1, n, n, Tl::TK, Tl::TJ, name);
  rc |= encode_3d_t(&maps[4], (const double*)u, n, n, Tl::TK, Tl::TJ, name);
  if (rc) return SGB_EINVAL;
  if (int rc = ensure_smem((const void*)star3_primal_f64_kernel<MODE>, Tl::SMEM, name))
    return rc;
  const int tiles_k = (int)((n + Tl::TK - 1) / Tl::TK);
  const long long tiles = (long long)tiles_k * ((n + Tl::TJ - 1) / Tl::TJ);
  const long long nout = hi - lo + 1;
  // wave model (two CTAs per SM) with ~48-plane chunks as the fp32 primal
  const long long slots = 2LL * num_sms();
  int nch = 1;
  long long best = -1;
  for (int cc = 1; cc <= 64 && cc <= nout; cc++) {
    const long long len = (nout + cc - 1) / cc;
    const long long cost = ((tiles * cc + slots - 1) / slots) * (len + 2 * R);
    if (best < 0 || cost < best) best = cost, nch = cc;
  }
  if (R >= 2) nch = (int)std::max<long long>(nch, (nout + 47) / 48);
  if (opt(OPT_PRIMAL_CHUNKS, 0) > 0) nch = (int)opt(OPT_PRIMAL_CHUNKS, 0);
  const int chunk = (int)((nout + nch - 1) / nch);
  const unsigned gy = (unsigned)((nout + chunk - 1) / chunk);
  star3_primal_f64_kernel<MODE><<<dim3((unsigned)tiles, gy), Tl::THREADS, Tl::SMEM, s>>>(
      maps[0], maps[1], maps[2], maps[3], maps[4], u, (int)n, (int)lo, (int)hi, chunk, tiles_k,
      D);
  return launch_status(name);
}

}  // namespace sgb
