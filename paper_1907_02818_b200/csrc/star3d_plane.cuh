// Plane-streaming gather adjoint for the 3D star families, any element type
// (the fp64 path, and fp32 shapes the TMA kernels do not take).
//
// Same predicate form of the reference's program as every gather kernel here
// (a term l reaches y iff y - o_l in B; adjoint.cpp:73-163,
// interp.cpp:189-198), organised like the fp32 streaming kernels but with
// plain loads: a CTA owns a 32 (k) x 8 (j) column tile and walks a chunk of
// output planes; per input plane p it stages the u_1 halo box and the masked
// q = D c^(1|2) u_b box (x in B) in shared memory, each thread forms the
// in-plane parts of Lap(u_1) and of the q-stencil for its point, and the i
// direction lives in 2R+1 rotating registers (plane loop unrolled by 2R+1).
// When plane p = o + R has been read, output plane o is complete:
//   u_1_b[o] += sum_l w_l q(o - o_l) + 2 u_b[o] [o in B]
//   c_b[o]   += S_c(o) u_b[o] [o in B],   u_2_b[o] -= u_b[o] [o in B] (c / c2)
// Points no term reaches are not written (their bits survive).
#pragma once

#include "generic_kernels.cuh"
#include "star3d_tma.cuh"

namespace sgb {

template <int MODE>
struct PlaneTile {
  static constexpr int R = Star3<MODE>::R;
  static constexpr int TK = 32, TJ = 8;
  static constexpr int BK = TK + 2 * R, BJ = TJ + 2 * R;
  static constexpr int RING = 2 * R + 1;
  static constexpr int THREADS = TK * TJ;
  static constexpr int BOX = BK * BJ;
  static constexpr int EPT = (BOX + THREADS - 1) / THREADS;
};

template <int MODE, typename T>
__global__ void __launch_bounds__(PlaneTile<MODE>::THREADS)
    star3_plane_kernel(Slab3 g, int lo, int hi, int out_i0, int out_i1, int chunk, T D,
                       const T* __restrict__ c, T* __restrict__ c_b, const T* __restrict__ u_1,
                       T* __restrict__ u_1_b, T* __restrict__ u_2_b,
                       const T* __restrict__ u_b) {
  using Tl = PlaneTile<MODE>;
  using S = Star3<MODE>;
  constexpr int R = Tl::R, BK = Tl::BK, RING = Tl::RING, TK = Tl::TK;
  __shared__ T U[Tl::BOX], Q[Tl::BOX];

  const int n = (int)g.n;
  const int tx = threadIdx.x % TK, ty = threadIdx.x / TK;
  const int k0 = blockIdx.x * TK, j0 = blockIdx.y * Tl::TJ;
  const int k = k0 + tx, j = j0 + ty;
  const int o_begin = out_i0 + blockIdx.z * chunk;
  const int o_end = min(o_begin + chunk, out_i1);
  if (o_begin >= o_end) return;
  const int pstart = o_begin - R;
  const int P = (o_end - o_begin) + 2 * R;
  const long long plane = (long long)n * n;

  T w[R + 1];
#pragma unroll
  for (int r = 0; r <= R; r++) w[r] = S::template w<T>(r);
  const int jout = j < lo ? lo - j : (j > hi ? j - hi : 0);
  const int kout = k < lo ? lo - k : (k > hi ? k - hi : 0);
  const bool own = j < n && k < n;
  const int sc = (ty + R) * BK + tx + R;  // this point in the box

  // box element offsets of this thread (fixed over planes)
  int boff[Tl::EPT], bgoff[Tl::EPT];
  bool bin[Tl::EPT], bB[Tl::EPT];
#pragma unroll
  for (int m = 0; m < Tl::EPT; m++) {
    const int e = threadIdx.x + m * Tl::THREADS;
    const int row = e / BK, col = e - (e / BK) * BK;
    const int jg = j0 - R + row, kg = k0 - R + col;
    boff[m] = e < Tl::BOX ? e : -1;
    bin[m] = e < Tl::BOX && jg >= 0 && jg < n && kg >= 0 && kg < n;
    bB[m] = jg >= lo && jg <= hi && kg >= lo && kg <= hi;
    bgoff[m] = bin[m] ? jg * n + kg : 0;
  }

  T al[RING], aq[RING];
#pragma unroll
  for (int s = 0; s < RING; s++) al[s] = aq[s] = T(0);

  for (int base = 0; base < P; base += RING) {
#pragma unroll
    for (int ph = 0; ph < RING; ph++) {
      const int it = base + ph;
      if (it < P) {
        const int p = pstart + it;
        const bool pin = p >= 0 && p < n;
        const bool pB = p >= lo && p <= hi;
        const long long pl = (long long)(p - (int)g.i_base) * plane;
#pragma unroll
        for (int m = 0; m < Tl::EPT; m++) {
          if (boff[m] >= 0) {
            T uv = T(0), qv = T(0);
            if (pin && bin[m]) {
              const long long x = pl + bgoff[m];
              uv = u_1[x];
              if (pB && bB[m]) {
                const T cv = c[x];
                qv = D * (S::kC2 ? cv * cv : cv) * u_b[x];
              }
            }
            U[boff[m]] = uv;
            Q[boff[m]] = qv;
          }
        }
        __syncthreads();
        // in-plane (j, k) parts at this point; centre values to the i ring
        const T uc = U[sc], qc = Q[sc];
        T li = w[0] * uc, qi = w[0] * qc;
#pragma unroll
        for (int r = 1; r <= R; r++) {
          li += w[r] * (U[sc - r] + U[sc + r] + U[sc - r * BK] + U[sc + r * BK]);
          qi += w[r] * (Q[sc - r] + Q[sc + r] + Q[sc - r * BK] + Q[sc + r * BK]);
        }
        al[ph] += li;
        aq[ph] += qi;
        al[(ph + R) % RING] = w[R] * uc;
        aq[(ph + R) % RING] = w[R] * qc;
#pragma unroll
        for (int r = 1; r <= R; r++) {
          if (r < R) {
            al[(ph + r) % RING] += w[r] * uc;
            aq[(ph + r) % RING] += w[r] * qc;
          }
          al[(ph + RING - r) % RING] += w[r] * uc;
          aq[(ph + RING - r) % RING] += w[r] * qc;
        }
        if (it >= 2 * R && own) {
          const int es = (ph + R + 1) % RING;
          const int o = p - R;
          const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
          const int nout = (oout > 0) + (jout > 0) + (kout > 0);
          const bool reach = nout == 0 || (nout == 1 && oout <= R && jout <= R && kout <= R);
          if (reach) {
            const long long y = (long long)(o - (int)g.i_base) * plane + (long long)j * n + k;
            const bool inB = nout == 0;
            T add = aq[es];
            if (inB) {
              const T ub = u_b[y];
              add += T(2) * ub;
              const T cv = c[y];
              const T scv = S::kC2 ? T(2) * D * cv : D;
              c_b[y] += scv * al[es] * ub;
              if (S::kU2) u_2_b[y] += -ub;
            }
            u_1_b[y] += add;
          }
        }
        __syncthreads();  // box consumed before the next plane's fill
      }
    }
  }
}

template <int MODE, typename T>
inline int star3_plane_gather(const Slab3& g, long long lo, long long hi, long long out_i0,
                              long long out_i1, T D, const T* c, T* c_b, const T* u_1,
                              T* u_1_b, T* u_2_b, const T* u_b, cudaStream_t s,
                              const char* name) {
  using Tl = PlaneTile<MODE>;
  const long long nout = out_i1 - out_i0;
  // ~256 output planes per CTA (measured insensitive: 64..768 within 4%); 2R halo planes
  // re-read per chunk (L2 hits for the most part)
  long long len = 256;
  if (opt(OPT_PLANE_CHUNK, 0) > 0) len = (int)opt(OPT_PLANE_CHUNK, 0);
  const int chunk = (int)std::min<long long>(nout, len);
  dim3 grid((unsigned)((g.n + Tl::TK - 1) / Tl::TK), (unsigned)((g.n + Tl::TJ - 1) / Tl::TJ),
            (unsigned)((nout + chunk - 1) / chunk));
  star3_plane_kernel<MODE, T><<<grid, Tl::THREADS, 0, s>>>(
      g, (int)lo, (int)hi, (int)out_i0, (int)out_i1, chunk, D, c, c_b, u_1, u_1_b, u_2_b, u_b);
  return launch_status(name);
}

// ---------------------------------------------------------------------------
// TMA-fed variant (default when n * sizeof(T) is a multiple of 16 and the
// arrays are 16-byte aligned): per input plane p one thread issues 3D TMA
// loads of the u_1 / c / u_b halo boxes of p and of the c, u_b, c_b, u_1_b
// tiles of the output plane o = p - R into a 3-stage mbarrier ring, so the
// loads run NS-1 planes ahead of the compute and out-of-grid / out-of-slab
// elements arrive as zeros; q = D c^(1|2) u_b [x in B] is formed in one shared
// pass.  Same arithmetic per point as star3_plane_kernel (bitwise equal).
template <int MODE, typename T>
struct PlaneTmaTile {
  static constexpr int R = Star3<MODE>::R;
  static constexpr int TK = 32, TJ = 8;
  static constexpr int BK = TK + 2 * R, BJ = TJ + 2 * R;
  static constexpr int RING = 2 * R + 1;
  static constexpr int NS = 3;
  static constexpr int THREADS = TK * TJ;
  static constexpr int BOX = BK * BJ, TILE = TK * TJ;
  // box slot stride: every TMA destination 128-byte aligned (radius 1: 34 x 10)
  static constexpr int BP = ((BOX * (int)sizeof(T) + 127) / 128) * 128 / (int)sizeof(T);
  static constexpr int EPT = (BOX + THREADS - 1) / THREADS;
  // stage: [u_1 box | c box | u_b box | c tile | u_b tile | c_b tile | u_1_b tile]
  static constexpr int SF = 3 * BP + 4 * TILE;
  static constexpr int SMEM = (NS * SF + BP) * (int)sizeof(T) + NS * 8;
  static_assert(RING % NS == 0, "static stage index");
  static constexpr bool kTmaRows = (BK * sizeof(T)) % 16 == 0 && (TK * sizeof(T)) % 16 == 0;
};

template <int MODE, typename T>
__global__ void __launch_bounds__(PlaneTmaTile<MODE, T>::THREADS)
    star3_plane_tma_kernel(const __grid_constant__ CUtensorMap tm_u1,
                           const __grid_constant__ CUtensorMap tm_c,
                           const __grid_constant__ CUtensorMap tm_ub,
                           const __grid_constant__ CUtensorMap tm_ct,
                           const __grid_constant__ CUtensorMap tm_ubt,
                           const __grid_constant__ CUtensorMap tm_cbt,
                           const __grid_constant__ CUtensorMap tm_u1bt, Slab3 g, int lo, int hi,
                           int out_i0, int out_i1, int chunk, T D, T* __restrict__ c_b,
                           T* __restrict__ u_1_b, T* __restrict__ u_2_b) {
  using Tl = PlaneTmaTile<MODE, T>;
  using S = Star3<MODE>;
  constexpr int R = Tl::R, BK = Tl::BK, RING = Tl::RING, TK = Tl::TK, NS = Tl::NS;
  constexpr int BOX = Tl::BOX, BP = Tl::BP, TILE = Tl::TILE, SF = Tl::SF;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* stage = reinterpret_cast<T*>(smem_raw);
  T* Q = stage + NS * SF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(Q + BP);

  const int n = (int)g.n;
  const int tid = threadIdx.x;
  const int tx = tid % TK, ty = tid / TK;
  const int k0 = blockIdx.x * TK, j0 = blockIdx.y * Tl::TJ;
  const int k = k0 + tx, j = j0 + ty;
  const int o_begin = out_i0 + blockIdx.z * chunk;
  const int o_end = min(o_begin + chunk, out_i1);
  if (o_begin >= o_end) return;
  const int pstart = o_begin - R;
  const int P = (o_end - o_begin) + 2 * R;
  const long long plane = (long long)n * n;

  T w[R + 1];
#pragma unroll
  for (int r = 0; r <= R; r++) w[r] = S::template w<T>(r);
  const int jout = j < lo ? lo - j : (j > hi ? j - hi : 0);
  const int kout = k < lo ? lo - k : (k > hi ? k - hi : 0);
  const bool own = j < n && k < n;
  const int sc = (ty + R) * BK + tx + R;
  const int st = ty * TK + tx;  // this point in a tile

  int boff[Tl::EPT];
  bool bB[Tl::EPT];
#pragma unroll
  for (int m = 0; m < Tl::EPT; m++) {
    const int e = tid + m * Tl::THREADS;
    const int row = e / BK, col = e - (e / BK) * BK;
    const int jg = j0 - R + row, kg = k0 - R + col;
    boff[m] = e < BOX ? e : -1;
    bB[m] = jg >= lo && jg <= hi && kg >= lo && kg <= hi;
  }

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int it) {
    const int s = it % NS;
    T* dst = stage + s * SF;
    const int pl = pstart + it - (int)g.i_base;
    const bool emit = it >= 2 * R;
    tma::mbar_arrive_expect_tx(&bars[s], (3 * BOX + (emit ? 4 * TILE : 0)) * (int)sizeof(T));
    tma::load_3d(dst, &tm_u1, &bars[s], k0 - R, j0 - R, pl);
    tma::load_3d(dst + BP, &tm_c, &bars[s], k0 - R, j0 - R, pl);
    tma::load_3d(dst + 2 * BP, &tm_ub, &bars[s], k0 - R, j0 - R, pl);
    if (emit) {
      const int ol = pl - R;
      tma::load_3d(dst + 3 * BP, &tm_ct, &bars[s], k0, j0, ol);
      tma::load_3d(dst + 3 * BP + TILE, &tm_ubt, &bars[s], k0, j0, ol);
      tma::load_3d(dst + 3 * BP + 2 * TILE, &tm_cbt, &bars[s], k0, j0, ol);
      tma::load_3d(dst + 3 * BP + 3 * TILE, &tm_u1bt, &bars[s], k0, j0, ol);
    }
  };
  if (tid == 0)
    for (int it = 0; it < NS && it < P; it++) issue(it);

  T al[RING], aq[RING];
#pragma unroll
  for (int s = 0; s < RING; s++) al[s] = aq[s] = T(0);

  for (int base = 0; base < P; base += RING) {
    const int par0 = base / NS;
#pragma unroll
    for (int ph = 0; ph < RING; ph++) {
      const int it = base + ph;
      if (it < P) {
        const int s = ph % NS;
        const int p = pstart + it;
        const T* U = stage + s * SF;
        const T* Cb = U + BP;
        const T* Ub = U + 2 * BP;
        tma::mbar_wait(&bars[s], (par0 + ph / NS) & 1);
        const bool pB = p >= lo && p <= hi;
#pragma unroll
        for (int m = 0; m < Tl::EPT; m++) {
          if (boff[m] >= 0) {
            T qv = T(0);
            if (pB && bB[m]) {
              const T cv = Cb[boff[m]];
              qv = D * (S::kC2 ? cv * cv : cv) * Ub[boff[m]];
            }
            Q[boff[m]] = qv;
          }
        }
        __syncthreads();
        const T uc = U[sc], qc = Q[sc];
        T li = w[0] * uc, qi = w[0] * qc;
#pragma unroll
        for (int r = 1; r <= R; r++) {
          li += w[r] * (U[sc - r] + U[sc + r] + U[sc - r * BK] + U[sc + r * BK]);
          qi += w[r] * (Q[sc - r] + Q[sc + r] + Q[sc - r * BK] + Q[sc + r * BK]);
        }
        al[ph] += li;
        aq[ph] += qi;
        al[(ph + R) % RING] = w[R] * uc;
        aq[(ph + R) % RING] = w[R] * qc;
#pragma unroll
        for (int r = 1; r <= R; r++) {
          if (r < R) {
            al[(ph + r) % RING] += w[r] * uc;
            aq[(ph + r) % RING] += w[r] * qc;
          }
          al[(ph + RING - r) % RING] += w[r] * uc;
          aq[(ph + RING - r) % RING] += w[r] * qc;
        }
        if (it >= 2 * R && own) {
          const int es = (ph + R + 1) % RING;
          const int o = p - R;
          const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
          const int nout = (oout > 0) + (jout > 0) + (kout > 0);
          const bool reach = nout == 0 || (nout == 1 && oout <= R && jout <= R && kout <= R);
          if (reach) {
            const T* tiles = U + 3 * BP;
            const long long y = (long long)(o - (int)g.i_base) * plane + (long long)j * n + k;
            const bool inB = nout == 0;
            T add = aq[es];
            if (inB) {
              const T ub = tiles[TILE + st];
              add += T(2) * ub;
              const T cv = tiles[st];
              const T scv = S::kC2 ? T(2) * D * cv : D;
              c_b[y] = tiles[2 * TILE + st] + scv * al[es] * ub;
              if (S::kU2) u_2_b[y] += -ub;
            }
            u_1_b[y] = tiles[3 * TILE + st] + add;
          }
        }
        __syncthreads();  // stage s and Q consumed
        if (tid == 0 && it + NS < P) issue(it + NS);
      }
    }
  }
}

template <typename T>
inline int encode_3d_t(CUtensorMap* map, const T* base, long long n, long long nplanes, int box0,
                       int box1, const char* name) {
  auto encode = get_encode();
  if (!encode) {
    set_error(std::string(name) + ": cuTensorMapEncodeTiled unavailable");
    return SGB_EINVAL;
  }
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)nplanes};
  cuuint64_t strides[2] = {(cuuint64_t)n * sizeof(T), (cuuint64_t)n * n * sizeof(T)};
  cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map,
                      sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                     : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                      3, (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(),
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(std::string(name) + ": tensor map encode failed (" + std::to_string((int)r) + ")");
    return SGB_EINVAL;
  }
  return 0;
}

// returns 1 when the TMA variant does not apply (caller uses the plain one)
template <int MODE, typename T>
inline int star3_plane_tma_gather(const Slab3& g, long long lo, long long hi, long long out_i0,
                                  long long out_i1, T D, const T* c, T* c_b, const T* u_1,
                                  T* u_1_b, T* u_2_b, const T* u_b, cudaStream_t s,
                                  const char* name) {
  using Tl = PlaneTmaTile<MODE, T>;
  if constexpr (!Tl::kTmaRows) {
    return 1;  // box rows not a 16-byte multiple (radius 1): plain-load kernel
  } else {
  if ((g.n * (long long)sizeof(T)) % 16 != 0 || g.n > (1 << 20)) return 1;
  for (const void* p : {(const void*)c, (const void*)c_b, (const void*)u_1, (const void*)u_1_b,
                        (const void*)u_b})
    if (reinterpret_cast<uintptr_t>(p) & 15) return 1;
  CUtensorMap maps[7];
  int rc = 0;
  rc |= encode_3d_t(&maps[0], u_1, g.n, g.nplanes, Tl::BK, Tl::BJ, name);
  rc |= encode_3d_t(&maps[1], c, g.n, g.nplanes, Tl::BK, Tl::BJ, name);
  rc |= encode_3d_t(&maps[2], u_b, g.n, g.nplanes, Tl::BK, Tl::BJ, name);
  rc |= encode_3d_t(&maps[3], c, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  rc |= encode_3d_t(&maps[4], u_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  rc |= encode_3d_t(&maps[5], (const T*)c_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  rc |= encode_3d_t(&maps[6], (const T*)u_1_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  if (rc) return SGB_EINVAL;
  if (int rc = ensure_smem((const void*)star3_plane_tma_kernel<MODE, T>, Tl::SMEM, name))
    return rc;
  const long long nout = out_i1 - out_i0;
  long long len = 256;
  if (opt(OPT_PLANE_CHUNK, 0) > 0) len = (int)opt(OPT_PLANE_CHUNK, 0);
  const int chunk = (int)std::min<long long>(nout, len);
  dim3 grid((unsigned)((g.n + Tl::TK - 1) / Tl::TK), (unsigned)((g.n + Tl::TJ - 1) / Tl::TJ),
            (unsigned)((nout + chunk - 1) / chunk));
  star3_plane_tma_kernel<MODE, T><<<grid, Tl::THREADS, Tl::SMEM, s>>>(
      maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], g, (int)lo, (int)hi,
      (int)out_i0, (int)out_i1, chunk, D, c_b, u_1_b, u_2_b);
  return launch_status(name);
  }
}

}  // namespace sgb
