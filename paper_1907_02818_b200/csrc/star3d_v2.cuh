// Streaming gather-adjoint kernel v2 for the 3D star families (sm_100a).
//
// Same mathematics and boundary predicate as star3d_tma.cuh (see the header
// comment there), re-balanced for B200:
//   * warp specialisation by field: warps [0, W/2) carry the Lap(u_1)
//     accumulators and emit c_b; warps [W/2, W) carry the q-stencil
//     accumulators and emit u_1_b (and u_2_b).  Each thread owns 2 rows x 4
//     consecutive k points, so per thread only one field's 2R+1 rotating
//     i-accumulators are live (2 x (2R+1) float4);
//   * 2-row register blocking cuts the j-direction shared-memory reads to
//     (2R + 2) 128-bit loads per 8 points and field;
//   * packed fp32x2 arithmetic (FFMA2 / FMUL2 / FADD2, sm_100) for every
//     operation that is lane-aligned;
//   * all point masks (j/k box membership, D folded in) precomputed once per
//     thread; only the plane predicate is evaluated per plane;
//   * adjoint read-modify-write with streaming (.cs) hints so L2 keeps the
//     input halos that neighbouring CTAs re-read.
#pragma once

#include <type_traits>

#include "star3d_tma.cuh"

namespace sgb {

__device__ __forceinline__ float2 lo2(const float4& v) { return make_float2(v.x, v.y); }
__device__ __forceinline__ float2 hi2(const float4& v) { return make_float2(v.z, v.w); }
__device__ __forceinline__ float4 cat4(const float2& a, const float2& b) {
  return make_float4(a.x, a.y, b.x, b.y);
}
// a*b + c on float4 via two FFMA2
__device__ __forceinline__ float4 fma4(const float4& a, const float4& b, const float4& c) {
  return cat4(__ffma2_rn(lo2(a), lo2(b), lo2(c)), __ffma2_rn(hi2(a), hi2(b), hi2(c)));
}
__device__ __forceinline__ float4 fmas4(float w, const float4& b, const float4& c) {
  const float2 ww = make_float2(w, w);
  return cat4(__ffma2_rn(ww, lo2(b), lo2(c)), __ffma2_rn(ww, hi2(b), hi2(c)));
}
__device__ __forceinline__ float4 mul4(const float4& a, const float4& b) {
  return cat4(__fmul2_rn(lo2(a), lo2(b)), __fmul2_rn(hi2(a), hi2(b)));
}
__device__ __forceinline__ float4 muls4(float w, const float4& b) {
  const float2 ww = make_float2(w, w);
  return cat4(__fmul2_rn(ww, lo2(b)), __fmul2_rn(ww, hi2(b)));
}
__device__ __forceinline__ float4 add4(const float4& a, const float4& b) {
  return cat4(__fadd2_rn(lo2(a), lo2(b)), __fadd2_rn(hi2(a), hi2(b)));
}
__device__ __forceinline__ float4 lds4(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

template <int MODE, int TJ_>
struct StarTile2 {
  static constexpr int R = Star3<MODE>::R;
  static constexpr int TK = 64, TJ = TJ_, HK = 4, HJ = R;
  static constexpr int BW = TK + 2 * HK;  // 72 floats
  static constexpr int BJ = TJ + 2 * HJ;
  static constexpr int RING = 2 * R + 1;
  static constexpr int ROLE = 16 * (TJ / 2);  // threads per role
  static constexpr int THREADS = 2 * ROLE;
  static constexpr int STAGES = 3;
  static constexpr int BOX_BYTES = BW * BJ * 4;
  static constexpr int FIELD_FLOATS = ((BOX_BYTES + 127) / 128) * 128 / 4;
  static constexpr int QUEUE = R + 1;
  static constexpr int QELEMS = (BW / 4) * BJ;  // float4 elements per box
  static constexpr int EPT = (QELEMS + THREADS - 1) / THREADS;
  static constexpr size_t SMEM = (size_t)(STAGES * 3 + 2) * FIELD_FLOATS * 4 +
                                 (size_t)QUEUE * ROLE * 2 * 16 + STAGES * 8;
  static constexpr int MIN_BLOCKS = THREADS <= 256 ? 2 : 1;
};

// k-direction part of the in-plane stencil for the 4 points of one row:
// window w[0..11] holds k0-4 .. k0+7 (centre points are w[4..7]).
template <int R>
__device__ __forceinline__ float4 kstencil(const float4& a, const float4& b, const float4& c,
                                           float w0, const float (&wr)[R + 1]) {
  const float w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
  float o[4];
#pragma unroll
  for (int m = 0; m < 4; m++) {
    float s = w0 * w[4 + m];
#pragma unroll
    for (int r = 1; r <= R; r++) s = fmaf(wr[r], w[4 + m - r] + w[4 + m + r], s);
    o[m] = s;
  }
  return make_float4(o[0], o[1], o[2], o[3]);
}

// One field's per-plane work for a 2-row x 4-point thread block: in-plane
// k/j stencil into acc[ph][row], centre values into the i neighbours.
template <int R, int RING>
__device__ __forceinline__ void field2(const float* F, int r0, int col, float w0,
                                       const float (&wr)[R + 1], float4 (&acc)[RING][2],
                                       int ph) {
  constexpr int BW = 72;
  const float* row0 = F + r0 * BW + col;  // centre float4 of row r0
  const float4 a0 = lds4(row0 - 4), b0 = lds4(row0), c0 = lds4(row0 + 4);
  const float4 a1 = lds4(row0 + BW - 4), b1 = lds4(row0 + BW), c1 = lds4(row0 + BW + 4);
  float4 in0 = kstencil<R>(a0, b0, c0, w0, wr);
  float4 in1 = kstencil<R>(a1, b1, c1, w0, wr);
  // j direction: the two centre rows feed each other at distance 1
  in0 = fmas4(wr[1], b1, in0);
  in1 = fmas4(wr[1], b0, in1);
#pragma unroll
  for (int t = -R; t <= R + 1; t++) {  // rows r0 + t, excluding the centre rows
    if (t == 0 || t == 1) continue;
    const float4 v = lds4(row0 + t * BW);
    const int d0 = t < 0 ? -t : t, d1 = (t - 1) < 0 ? 1 - t : t - 1;
    if (d0 <= R) in0 = fmas4(wr[d0], v, in0);
    if (d1 <= R) in1 = fmas4(wr[d1], v, in1);
  }
  acc[ph][0] = add4(acc[ph][0], in0);
  acc[ph][1] = add4(acc[ph][1], in1);
  // i direction; output p+R gets its first contribution here (initialise)
  acc[(ph + R) % RING][0] = muls4(wr[R], b0);
  acc[(ph + R) % RING][1] = muls4(wr[R], b1);
#pragma unroll
  for (int r = 1; r <= R; r++) {
    if (r < R) {
      acc[(ph + r) % RING][0] = fmas4(wr[r], b0, acc[(ph + r) % RING][0]);
      acc[(ph + r) % RING][1] = fmas4(wr[r], b1, acc[(ph + r) % RING][1]);
    }
    acc[(ph + RING - r) % RING][0] = fmas4(wr[r], b0, acc[(ph + RING - r) % RING][0]);
    acc[(ph + RING - r) % RING][1] = fmas4(wr[r], b1, acc[(ph + RING - r) % RING][1]);
  }
}

__device__ __forceinline__ float4 sel4(const bool (&m)[4], const float4& yes, const float4& no) {
  return make_float4(m[0] ? yes.x : no.x, m[1] ? yes.y : no.y, m[2] ? yes.z : no.z,
                     m[3] ? yes.w : no.w);
}

template <int MODE, int TJ>
__global__ void __launch_bounds__(StarTile2<MODE, TJ>::THREADS, StarTile2<MODE, TJ>::MIN_BLOCKS)
    star3_v2_kernel(const __grid_constant__ CUtensorMap tm_c,
                    const __grid_constant__ CUtensorMap tm_ub,
                    const __grid_constant__ CUtensorMap tm_u1, float* __restrict__ c_b,
                    float* __restrict__ u_1_b, float* __restrict__ u_2_b, int n, int i_base,
                    int lo, int hi, int out_i0, int out_i1, int chunk, int tiles_k, float D) {
  using Tl = StarTile2<MODE, TJ>;
  using S3 = Star3<MODE>;
  constexpr int R = Tl::R, HJ = Tl::HJ, HK = Tl::HK, BW = Tl::BW;
  constexpr int RING = Tl::RING, NS = Tl::STAGES, FW = Tl::FIELD_FLOATS, QD = Tl::QUEUE;
  constexpr int ROLE = Tl::ROLE, EPT = Tl::EPT;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);
  float* qbuf = stage + NS * 3 * FW;
  float4* gq = reinterpret_cast<float4*>(qbuf + 2 * FW);  // [QD][ROLE][2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(gq + QD * ROLE * 2);

  const int tid = threadIdx.x;
  const bool lap_role = tid < ROLE;  // warp-uniform (ROLE is a multiple of 32)
  const int rt = lap_role ? tid : tid - ROLE;
  const int tx = rt & 15, ty = rt >> 4;
  const int tk = blockIdx.x % tiles_k, tj = blockIdx.x / tiles_k;
  const int k0 = tk * Tl::TK, j0 = tj * Tl::TJ;
  const int o_begin = out_i0 + blockIdx.y * chunk;
  const int o_end = min(o_begin + chunk, out_i1);
  if (o_begin >= o_end) return;
  const int pstart = o_begin - R;
  const int P = (o_end - o_begin) + 2 * R;

  const float w0 = S3::template w<float>(0);
  float wr[R + 1];
  wr[0] = w0;
#pragma unroll
  for (int r = 1; r <= R; r++) wr[r] = S3::template w<float>(r);

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; s++) tma::mbar_init(&bars[s], 1);
    tma::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int it) {
    const int s = it % NS;
    float* dst = stage + s * 3 * FW;
    const int pl = pstart + it - i_base;
    tma::mbar_arrive_expect_tx(&bars[s], 3 * Tl::BOX_BYTES);
    tma::load_3d(dst + 0 * FW, &tm_c, &bars[s], k0 - HK, j0 - HJ, pl);
    tma::load_3d(dst + 1 * FW, &tm_ub, &bars[s], k0 - HK, j0 - HJ, pl);
    tma::load_3d(dst + 2 * FW, &tm_u1, &bars[s], k0 - HK, j0 - HJ, pl);
  };
  if (tid == 0)
    for (int it = 0; it < NS && it < P; it++) issue(it);

  // ---- this thread's 2 x 4 output points
  const int jr0 = j0 + 2 * ty;
  const int kc = k0 + 4 * tx;
  const int r0 = 2 * ty + HJ;   // box row of jr0
  const int col = HK + 4 * tx;  // box column of kc
  const long long plane = (long long)n * n;
  const long long coff0 = (long long)jr0 * n + kc;
  // A block is "interior" when its whole halo box lies inside [lo, hi] in j and
  // k: then every j/k mask is 1 and only the per-plane predicates remain.
  const bool interior = j0 - HJ >= lo && j0 + Tl::TJ + HJ - 1 <= hi && k0 - HK >= lo &&
                        k0 + Tl::TK + HK - 1 <= hi && j0 + Tl::TJ <= n && k0 + Tl::TK <= n;

  float4 acc[RING][2];
#pragma unroll
  for (int s = 0; s < RING; s++) acc[s][0] = acc[s][1] = make_float4(0.f, 0.f, 0.f, 0.f);

  auto run = [&](auto interior_tag) {
    constexpr bool INT = decltype(interior_tag)::value;
    // j/k masks (boundary blocks only; constant-folded for interior blocks)
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
    auto kmask = [&](int h, float f) {  // f where (j,k) in B, else 0
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
          const float* Cs = stage + s * 3 * FW;
          const float* UBs = Cs + FW;
          const float* U1s = Cs + 2 * FW;
          float* Q = qbuf + (it & 1) * FW;
          const bool emit = it >= 2 * R;
          const int o = p - R;
          const bool pin = p >= lo && p <= hi;
          const bool oin = o >= lo && o <= hi;
          const long long obase = (long long)(o - i_base) * plane;

          // prefetch the adjoint values this plane's emit updates (streaming)
          float4 old[2] = {make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
          if (emit) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
              if (!rowok(h)) continue;
              const long long gi = obase + coff0 + (long long)h * n;
              if (lap_role) {
                if (oin && jin(h)) old[h] = __ldcs(reinterpret_cast<const float4*>(c_b + gi));
              } else {
                old[h] = __ldcs(reinterpret_cast<const float4*>(u_1_b + gi));
              }
            }
          }

          tma::mbar_wait(&bars[s], (it / NS) & 1);

          // ---- q = D c(^2) u_b [x in B] over the halo box
#pragma unroll
          for (int m = 0; m < EPT; m++) {
            const int e = tid + m * Tl::THREADS;
            if (e >= Tl::QELEMS) continue;
            const int row = e / (BW / 4), c4 = e - row * (BW / 4);
            const int qo = row * BW + 4 * c4;
            float4 qv = make_float4(0.f, 0.f, 0.f, 0.f);
            if (pin) {
              const float4 cv = lds4(Cs + qo);
              const float4 uv = lds4(UBs + qo);
              const float4 cq = S3::kC2 ? mul4(cv, cv) : cv;
              float4 dm = make_float4(D, D, D, D);
              if (!INT) {
                const int jg = j0 - HJ + row, kg = k0 - HK + 4 * c4;
                const bool rm = jg >= lo && jg <= hi;
                dm = make_float4((rm && kg >= lo && kg <= hi) ? D : 0.f,
                                 (rm && kg + 1 >= lo && kg + 1 <= hi) ? D : 0.f,
                                 (rm && kg + 2 >= lo && kg + 2 <= hi) ? D : 0.f,
                                 (rm && kg + 3 >= lo && kg + 3 <= hi) ? D : 0.f);
              }
              qv = mul4(mul4(cq, uv), dm);
            }
            *reinterpret_cast<float4*>(Q + qo) = qv;
          }
          // ---- per-role centre work for plane p
          if (lap_role) {
            // g = 2 D c u_b (c^2) or D u_b (linear), masked; queued R planes
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
          } else if (pin) {
            // u_1_b centre term 2 u_b (into this plane's accumulator) and, for
            // the c-modes, u_2_b += -u_b at this very plane
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
          __syncthreads();
          if (tid == 0 && it >= 1 && it - 1 + NS < P) issue(it - 1 + NS);

          // ---- stencils: Lap(u_1) on the Lap role, q stencil on the q role
          field2<R, RING>(lap_role ? U1s : Q, r0, col, w0, wr, acc, ph);

          // ---- emit output plane o = p - R
          if (emit) {
            const int es = (ph + R + 1) % RING;
            if (lap_role) {
              if (oin) {
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
              const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
#pragma unroll
              for (int h = 0; h < 2; h++) {
                if (!rowok(h)) continue;
                float4 nv;
                if (INT) {
                  if (oout > R) continue;  // plane not reached at all
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

template <int MODE, int TJ>
inline int star3_v2_gather(const Slab3& g, long long lo, long long hi, long long out_i0,
                           long long out_i1, float D, const float* c, float* c_b,
                           const float* u_1, float* u_1_b, float* u_2_b, const float* u_b,
                           cudaStream_t s, const char* name) {
  using Tl = StarTile2<MODE, TJ>;
  auto encode = get_encode();
  if (!encode) {
    set_error(std::string(name) + ": cuTensorMapEncodeTiled unavailable");
    return SGB_EINVAL;
  }
  CUtensorMap maps[3];
  const float* src[3] = {c, u_b, u_1};
  for (int f = 0; f < 3; f++) {
    cuuint64_t dims[3] = {(cuuint64_t)g.n, (cuuint64_t)g.n, (cuuint64_t)g.nplanes};
    cuuint64_t strides[2] = {(cuuint64_t)g.n * 4, (cuuint64_t)g.n * g.n * 4};
    cuuint32_t box[3] = {(cuuint32_t)Tl::BW, (cuuint32_t)Tl::BJ, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(&maps[f], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)src[f], dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(),
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error(std::string(name) + ": tensor map encode failed (" + std::to_string((int)r) +
                ")");
      return SGB_EINVAL;
    }
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(star3_v2_kernel<MODE, TJ>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Tl::SMEM);
    attr_set = true;
  }
  const int tiles_k = (int)((g.n + Tl::TK - 1) / Tl::TK);
  const int tiles_j = (int)((g.n + Tl::TJ - 1) / Tl::TJ);
  const long long nout = out_i1 - out_i0;
  const int chunks = choose_chunks((long long)tiles_k * tiles_j, nout, Tl::R, Tl::MIN_BLOCKS);
  const int chunk = (int)((nout + chunks - 1) / chunks);
  dim3 grid((unsigned)(tiles_k * tiles_j), (unsigned)((nout + chunk - 1) / chunk));
  star3_v2_kernel<MODE, TJ><<<grid, Tl::THREADS, Tl::SMEM, s>>>(
      maps[0], maps[1], maps[2], c_b, u_1_b, u_2_b, (int)g.n, (int)g.i_base, (int)lo, (int)hi,
      (int)out_i0, (int)out_i1, chunk, tiles_k, D);
  return launch_status(name);
}

}  // namespace sgb
