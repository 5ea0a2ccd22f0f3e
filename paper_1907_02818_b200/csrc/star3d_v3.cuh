// Streaming gather-adjoint kernel v3 for the 3D star families (sm_100a):
// warp-specialised, mbarrier-pipelined, no block-wide barrier in the loop.
//
// Mathematics and boundary predicate: as star3d_tma.cuh (
// reference adjoint.cpp:73-163, interp.cpp:189-198).
//
// Warp roles (one CTA = one 64 (k) x 16 (j) column tile, streaming over i):
//   warp 0          TMA issuer: per plane p, three halo boxes (c, u_b, u_1)
//                   and, for the output plane o = p - R, the two adjoint tiles
//                   (c_b, u_1_b) -- all cp.async.bulk.tensor into one stage of
//                   an NS-deep ring, completion via full[s] (expect_tx);
//                   refills a stage once empty[s] says every role is done;
//   warps 1..NP     q producers: q = D c(^2) u_b [x in B] for the halo box into
//                   an NQ-deep q ring (qfull / qempty mbarriers);
//   NL "Lap" warps  Lap(u_1) stencil + rotating i-accumulators; g = 2 D c u_b
//                   queued R planes; emit c_b[o] = old + g Lap;
//   NQW "q" warps   q stencil + 2 u_b centre term; emit u_1_b[o]; u_2_b[p].
// Each consumer thread owns 2 rows x 4 k-points; arithmetic is packed fp32x2.
// Consumers read the old adjoint values from shared memory (TMA-prefetched)
// and write results with streaming 128-bit stores, so no consumer ever waits
// on a global load.
#pragma once

#include <type_traits>

#include "star3d_v2.cuh"

namespace sgb {

namespace tma {
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
}  // namespace tma

template <int MODE>
struct StarTile3 {
  static constexpr int R = Star3<MODE>::R;
  static constexpr int TK = 64, TJ = 16, HK = 4, HJ = R;
  static constexpr int BW = TK + 2 * HK;  // 72
  static constexpr int BJ = TJ + 2 * HJ;
  static constexpr int RING = 2 * R + 1;
  static constexpr int NS = 4;  // TMA stages
  static constexpr int NQ = 3;  // q ring
  static constexpr int NPW = 2;  // q-producer warps
  static constexpr int NCW = 4;  // warps per consumer role (2 rows x 4 pts x 128 thr)
  static constexpr int THREADS = 32 * (1 + NPW + 2 * NCW);
  static constexpr int ROLE = NCW * 32;
  static constexpr int BOX_BYTES = BW * BJ * 4;
  static constexpr int BOX_FLOATS = ((BOX_BYTES + 127) / 128) * 128 / 4;
  static constexpr int TILE_BYTES = TK * TJ * 4;
  static constexpr int TILE_FLOATS = TK * TJ;
  static constexpr int STAGE_FLOATS = 3 * BOX_FLOATS + 2 * TILE_FLOATS;
  static constexpr int QUEUE = R + 1;
  static constexpr int QELEMS = (BW / 4) * BJ;
  static constexpr size_t SMEM = (size_t)NS * STAGE_FLOATS * 4 + (size_t)NQ * BOX_FLOATS * 4 +
                                 (size_t)QUEUE * ROLE * 2 * 16 + (2 * NS + 2 * NQ) * 8;
};

template <int MODE>
__global__ void __launch_bounds__(StarTile3<MODE>::THREADS, 1)
    star3_v3_kernel(const __grid_constant__ CUtensorMap tm_c,
                    const __grid_constant__ CUtensorMap tm_ub,
                    const __grid_constant__ CUtensorMap tm_u1,
                    const __grid_constant__ CUtensorMap tm_cb,
                    const __grid_constant__ CUtensorMap tm_u1b, float* __restrict__ c_b,
                    float* __restrict__ u_1_b, float* __restrict__ u_2_b, int n, int i_base,
                    int lo, int hi, int out_i0, int out_i1, int chunk, int tiles_k, float D) {
  using Tl = StarTile3<MODE>;
  using S3 = Star3<MODE>;
  constexpr int R = Tl::R, HJ = Tl::HJ, HK = Tl::HK, BW = Tl::BW, TK = Tl::TK;
  constexpr int RING = Tl::RING, NS = Tl::NS, NQ = Tl::NQ, QD = Tl::QUEUE;
  constexpr int BF = Tl::BOX_FLOATS, SF = Tl::STAGE_FLOATS, ROLE = Tl::ROLE;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);  // [NS][c, ub, u1, cb, u1b]
  float* qring = stage + NS * SF;                      // [NQ][box]
  float4* gq = reinterpret_cast<float4*>(qring + NQ * BF);  // [QD][ROLE][2]
  uint64_t* full = reinterpret_cast<uint64_t*>(gq + QD * ROLE * 2);
  uint64_t* empty = full + NS;
  uint64_t* qfull = empty + NS;
  uint64_t* qempty = qfull + NQ;

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int tk = blockIdx.x % tiles_k, tj = blockIdx.x / tiles_k;
  const int k0 = tk * TK, j0 = tj * Tl::TJ;
  const int o_begin = out_i0 + blockIdx.y * chunk;
  const int o_end = min(o_begin + chunk, out_i1);
  if (o_begin >= o_end) return;
  const int pstart = o_begin - R;
  const int P = (o_end - o_begin) + 2 * R;

  constexpr int NPROD = Tl::NPW * 32;
  constexpr int EMPTY_COUNT = NPROD + 2 * ROLE;
  if (tid == 0) {
    for (int s = 0; s < NS; s++) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], EMPTY_COUNT);
    }
    for (int q = 0; q < NQ; q++) {
      tma::mbar_init(&qfull[q], NPROD);
      tma::mbar_init(&qempty[q], ROLE);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();

  // ------------------------------------------------------------ TMA warp
  if (warp == 0) {
    if ((tid & 31) != 0) return;
    for (int it = 0; it < P; it++) {
      const int s = it % NS, k = it / NS;
      if (k > 0) tma::mbar_wait(&empty[s], (k - 1) & 1);
      float* dst = stage + s * SF;
      const int p = pstart + it;
      const int pl = p - i_base;
      const bool emit = it >= 2 * R;
      tma::mbar_arrive_expect_tx(&full[s], 3 * Tl::BOX_BYTES + (emit ? 2 * Tl::TILE_BYTES : 0));
      tma::load_3d(dst + 0 * BF, &tm_c, &full[s], k0 - HK, j0 - HJ, pl);
      tma::load_3d(dst + 1 * BF, &tm_ub, &full[s], k0 - HK, j0 - HJ, pl);
      tma::load_3d(dst + 2 * BF, &tm_u1, &full[s], k0 - HK, j0 - HJ, pl);
      if (emit) {
        tma::load_3d(dst + 3 * BF, &tm_cb, &full[s], k0, j0, pl - R);
        tma::load_3d(dst + 3 * BF + Tl::TILE_FLOATS, &tm_u1b, &full[s], k0, j0, pl - R);
      }
    }
    return;
  }

  // ------------------------------------------------------------ q producers
  if (warp <= Tl::NPW) {
    const int pt = tid - 32;
    for (int it = 0; it < P; it++) {
      const int s = it % NS;
      const int slot = it % NQ, kq = it / NQ;
      const int p = pstart + it;
      const bool pin = p >= lo && p <= hi;
      tma::mbar_wait(&full[s], (it / NS) & 1);
      if (kq > 0) tma::mbar_wait(&qempty[slot], (kq - 1) & 1);
      const float* Cs = stage + s * SF;
      const float* UBs = Cs + BF;
      float* Q = qring + slot * BF;
      for (int e = pt; e < Tl::QELEMS; e += NPROD) {
        const int row = e / (BW / 4), c4 = e - row * (BW / 4);
        const int qo = row * BW + 4 * c4;
        float4 qv = make_float4(0.f, 0.f, 0.f, 0.f);
        if (pin) {
          const int jg = j0 - HJ + row, kg = k0 - HK + 4 * c4;
          const bool rm = jg >= lo && jg <= hi;
          const float4 dm = make_float4((rm && kg >= lo && kg <= hi) ? D : 0.f,
                                        (rm && kg + 1 >= lo && kg + 1 <= hi) ? D : 0.f,
                                        (rm && kg + 2 >= lo && kg + 2 <= hi) ? D : 0.f,
                                        (rm && kg + 3 >= lo && kg + 3 <= hi) ? D : 0.f);
          const float4 cv = lds4(Cs + qo);
          const float4 uv = lds4(UBs + qo);
          qv = mul4(mul4(S3::kC2 ? mul4(cv, cv) : cv, uv), dm);
        }
        *reinterpret_cast<float4*>(Q + qo) = qv;
      }
      tma::mbar_arrive(&qfull[slot]);
      tma::mbar_arrive(&empty[s]);
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  const bool lap_role = warp < 1 + Tl::NPW + Tl::NCW;  // warp-uniform
  const int rt = tid - 32 * (1 + Tl::NPW) - (lap_role ? 0 : ROLE);
  const int tx = rt & 15, ty = rt >> 4;
  const int jr0 = j0 + 2 * ty;
  const int kc = k0 + 4 * tx;
  const int r0 = 2 * ty + HJ;   // box row of jr0
  const int col = HK + 4 * tx;  // box column of kc
  const int trow = 2 * ty * TK + 4 * tx;  // offset in the 64x16 adjoint tile
  const long long plane = (long long)n * n;
  const long long coff0 = (long long)jr0 * n + kc;
  const float w0 = S3::template w<float>(0);
  float wr[R + 1];
  wr[0] = w0;
#pragma unroll
  for (int r = 1; r <= R; r++) wr[r] = S3::template w<float>(r);
  const bool interior = j0 - HJ >= lo && j0 + Tl::TJ + HJ - 1 <= hi && k0 - HK >= lo &&
                        k0 + TK + HK - 1 <= hi && j0 + Tl::TJ <= n && k0 + TK <= n;

  float4 acc[RING][2];
#pragma unroll
  for (int s = 0; s < RING; s++) acc[s][0] = acc[s][1] = make_float4(0.f, 0.f, 0.f, 0.f);

  auto run = [&](auto interior_tag) {
    constexpr bool INT = decltype(interior_tag)::value;
    auto kin = [&](int m) { return INT || (kc + m >= lo && kc + m <= hi); };
    auto kout = [&](int m) {
      const int k = kc + m;
      return INT ? 0 : (k < lo ? lo - k : (k > hi ? k - hi : 0));
    };
    auto jin = [&](int h) { return INT || (jr0 + h >= lo && jr0 + h <= hi); };
    auto jout = [&](int h) {
      const int j = jr0 + h;
      return INT ? 0 : (j < lo ? lo - j : (j > hi ? j - hi : 0));
    };
    auto rowok = [&](int h) { return INT || (jr0 + h < n && kc < n); };
    auto kmask = [&](int h, float f) {
      if (INT) return make_float4(f, f, f, f);
      const bool jj = jin(h);
      return make_float4((jj && kin(0)) ? f : 0.f, (jj && kin(1)) ? f : 0.f,
                         (jj && kin(2)) ? f : 0.f, (jj && kin(3)) ? f : 0.f);
    };
    auto kinv = [&](bool (&m)[4]) {
#pragma unroll
      for (int q = 0; q < 4; q++) m[q] = kin(q);
    };

    for (int base = 0; base < P; base += RING) {
#pragma unroll
      for (int ph = 0; ph < RING; ph++) {
        const int it = base + ph;
        if (it < P) {
          const int s = it % NS;
          const int p = pstart + it;
          const float* Cs = stage + s * SF;
          const float* UBs = Cs + BF;
          const float* U1s = Cs + 2 * BF;
          const float* OLD = Cs + 3 * BF + (lap_role ? 0 : Tl::TILE_FLOATS);
          const bool emit = it >= 2 * R;
          const int o = p - R;
          const bool pin = p >= lo && p <= hi;
          const bool oin = o >= lo && o <= hi;
          const long long obase = (long long)(o - i_base) * plane;
          const int es = (ph + R + 1) % RING;

          tma::mbar_wait(&full[s], (it / NS) & 1);
          float4 old[2];
          old[0] = lds4(OLD + trow);
          old[1] = lds4(OLD + trow + TK);

          if (lap_role) {
            // g for plane p (queued R planes)
#pragma unroll
            for (int h = 0; h < 2; h++) {
              float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
              if (pin) {
                const float4 uv = lds4(UBs + (r0 + h) * BW + col);
                const float4 cm = kmask(h, S3::kC2 ? 2.f * D : D);
                if (S3::kC2) {
                  const float4 cv = lds4(Cs + (r0 + h) * BW + col);
                  g = mul4(mul4(cv, uv), cm);
                } else {
                  g = mul4(uv, cm);
                }
              }
              gq[((it % QD) * ROLE + rt) * 2 + h] = g;
            }
            field2<R, RING>(U1s, r0, col, w0, wr, acc, ph);
            tma::mbar_arrive(&empty[s]);
            if (emit && oin) {
#pragma unroll
              for (int h = 0; h < 2; h++) {
                if (!rowok(h) || !jin(h)) continue;
                const float4 g = gq[(((it - R) % QD) * ROLE + rt) * 2 + h];
                float4 nv = fma4(g, acc[es][h], old[h]);
                if (!INT) {
                  bool km[4];
                  kinv(km);
                  nv = sel4(km, nv, old[h]);
                }
                __stcs(reinterpret_cast<float4*>(c_b + obase + coff0 + (long long)h * n), nv);
              }
            }
          } else {
            const int slot = it % NQ;
            if (pin) {
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const float4 uv = lds4(UBs + (r0 + h) * BW + col);
                const float4 um = INT ? uv : mul4(uv, kmask(h, 1.f));
                acc[ph][h] = fmas4(2.f, um, acc[ph][h]);
                if (S3::kU2 && rowok(h) && jin(h) && p >= o_begin && p < o_end) {
                  float* ptr = u_2_b + (long long)(p - i_base) * plane + coff0 + (long long)h * n;
                  float4 u2 = __ldcs(reinterpret_cast<const float4*>(ptr));
                  bool km[4];
                  kinv(km);
                  u2 = sel4(km, add4(u2, make_float4(-um.x, -um.y, -um.z, -um.w)), u2);
                  __stcs(reinterpret_cast<float4*>(ptr), u2);
                }
              }
            }
            tma::mbar_arrive(&empty[s]);  // stage no longer read by this role
            tma::mbar_wait(&qfull[slot], (it / NQ) & 1);
            field2<R, RING>(qring + slot * BF, r0, col, w0, wr, acc, ph);
            tma::mbar_arrive(&qempty[slot]);
            if (emit) {
              const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
#pragma unroll
              for (int h = 0; h < 2; h++) {
                if (!rowok(h)) continue;
                float4 nv;
                if (INT) {
                  if (oout > R) continue;
                  nv = add4(old[h], acc[es][h]);
                } else {
                  bool reach[4];
#pragma unroll
                  for (int m = 0; m < 4; m++) {
                    const int nout = (oout > 0) + (jout(h) > 0) + (kout(m) > 0);
                    reach[m] =
                        nout == 0 || (nout == 1 && oout <= R && jout(h) <= R && kout(m) <= R);
                  }
                  nv = sel4(reach, add4(old[h], acc[es][h]), old[h]);
                }
                __stcs(reinterpret_cast<float4*>(u_1_b + obase + coff0 + (long long)h * n), nv);
              }
            }
          }
        }
      }
    }
  };
  if (interior)
    run(std::true_type{});
  else
    run(std::false_type{});
}

inline int encode_3d(CUtensorMap* map, const float* base, long long n, long long nplanes,
                     int box0, int box1, const char* name) {
  auto encode = get_encode();
  if (!encode) {
    set_error(std::string(name) + ": cuTensorMapEncodeTiled unavailable");
    return SGB_EINVAL;
  }
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)nplanes};
  cuuint64_t strides[2] = {(cuuint64_t)n * 4, (cuuint64_t)n * n * 4};
  cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)base, dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(std::string(name) + ": tensor map encode failed (" + std::to_string((int)r) + ")");
    return SGB_EINVAL;
  }
  return 0;
}

// Same, restricted to the window [off, off+ext) in j and k: TMA zero-fills
// every element outside it, which is exactly the primal-box mask on the seed
// (u_b is defined on [lo, hi]^3 only).  Needs a 16-byte aligned window base;
// returns 1 (no map) when it is not.
inline int encode_3d_window(CUtensorMap* map, const float* base, long long n, long long nplanes,
                            long long off, long long ext, int box0, int box1, const char* name) {
  const float* wb = base + off * n + off;
  if ((reinterpret_cast<uintptr_t>(wb) & 15) != 0 || ext < 1) return 1;
  auto encode = get_encode();
  if (!encode) {
    set_error(std::string(name) + ": cuTensorMapEncodeTiled unavailable");
    return SGB_EINVAL;
  }
  cuuint64_t dims[3] = {(cuuint64_t)ext, (cuuint64_t)ext, (cuuint64_t)nplanes};
  cuuint64_t strides[2] = {(cuuint64_t)n * 4, (cuuint64_t)n * n * 4};
  cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)wb, dims, strides, box,
                      estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error(std::string(name) + ": tensor map encode failed (" + std::to_string((int)r) + ")");
    return SGB_EINVAL;
  }
  return 0;
}

template <int MODE>
inline int star3_v3_gather(const Slab3& g, long long lo, long long hi, long long out_i0,
                           long long out_i1, float D, const float* c, float* c_b,
                           const float* u_1, float* u_1_b, float* u_2_b, const float* u_b,
                           cudaStream_t s, const char* name) {
  using Tl = StarTile3<MODE>;
  CUtensorMap maps[5];
  int rc = 0;
  rc |= encode_3d(&maps[0], c, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  rc |= encode_3d(&maps[1], u_b, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  rc |= encode_3d(&maps[2], u_1, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  rc |= encode_3d(&maps[3], c_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  rc |= encode_3d(&maps[4], u_1_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  if (rc) return SGB_EINVAL;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(star3_v3_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Tl::SMEM);
    attr_set = true;
  }
  const int tiles_k = (int)((g.n + Tl::TK - 1) / Tl::TK);
  const int tiles_j = (int)((g.n + Tl::TJ - 1) / Tl::TJ);
  const long long nout = out_i1 - out_i0;
  const int chunks = choose_chunks((long long)tiles_k * tiles_j, nout, Tl::R, 1);
  const int chunk = (int)((nout + chunks - 1) / chunks);
  dim3 grid((unsigned)(tiles_k * tiles_j), (unsigned)((nout + chunk - 1) / chunk));
  star3_v3_kernel<MODE><<<grid, Tl::THREADS, Tl::SMEM, s>>>(
      maps[0], maps[1], maps[2], maps[3], maps[4], c_b, u_1_b, u_2_b, (int)g.n, (int)g.i_base,
      (int)lo, (int)hi, (int)out_i0, (int)out_i1, chunk, tiles_k, D);
  return launch_status(name);
}

}  // namespace sgb
