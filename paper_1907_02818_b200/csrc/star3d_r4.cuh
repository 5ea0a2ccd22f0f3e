// Radius-4 streaming gather-adjoint kernel (the hot kernel; sm_100a).
//
// Mathematics and boundary predicate: star3d_tma.cuh header (SURVEY
// Appendix C; reference adjoint.cpp:73-163 / interp.cpp:189-198).  Design,
// measurements and the path from the earlier versions: DESIGN.md ("Radius-4
// streaming kernel") and profiles/.
//
// Instantiated for MODE 2 (wave3d_r4: the reference's wave3d_r4_b), MODE 3
// (the same plus the time-loop u_2 partial written from the u_b box the
// q-role threads already hold) and MODE 4 (u_1_b = this call's adjoint:
// zeroing fused, the u_1_b tile not loaded); MODE 0 / 1 (radius 1) compile
// too but the v1 kernel is faster there (star3d_tma.cuh).
#pragma once
#include <cstring>
#include <mutex>
#include <utility>

#include "star3d_tma.cuh"

namespace sgb {

// ---- packed fp32x2 helpers on float4 (FFMA2 / FMUL2 / FADD2)
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

__device__ __forceinline__ float4 sel4(const bool (&m)[4], const float4& yes, const float4& no) {
  return make_float4(m[0] ? yes.x : no.x, m[1] ? yes.y : no.y, m[2] ? yes.z : no.z,
                     m[3] ? yes.w : no.w);
}


// in-plane k-direction stencil for 4 points: window a|b|c = k0-4 .. k0+7
template <int R>
__device__ __forceinline__ float4 kstencil2(const float4& a, const float4& b, const float4& c,
                                            float w0, const float (&wr)[R + 1]) {
  const float w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
  float2 p0 = __fmul2_rn(make_float2(w0, w0), make_float2(w[4], w[5]));
  float2 p1 = __fmul2_rn(make_float2(w0, w0), make_float2(w[6], w[7]));
#pragma unroll
  for (int r = 1; r <= R; r++) {
    const float2 ww = make_float2(wr[r], wr[r]);
    if ((r & 1) == 0) {  // lane-aligned pairs
      p0 = __ffma2_rn(ww, __fadd2_rn(make_float2(w[4 - r], w[5 - r]), make_float2(w[4 + r], w[5 + r])), p0);
      p1 = __ffma2_rn(ww, __fadd2_rn(make_float2(w[6 - r], w[7 - r]), make_float2(w[6 + r], w[7 + r])), p1);
    } else {
      const float s0 = w[4 - r] + w[4 + r], s1 = w[5 - r] + w[5 + r];
      const float s2 = w[6 - r] + w[6 + r], s3 = w[7 - r] + w[7 + r];
      p0 = __ffma2_rn(ww, make_float2(s0, s1), p0);
      p1 = __ffma2_rn(ww, make_float2(s2, s3), p1);
    }
  }
  return cat4(p0, p1);
}

// ---- 3D tensor maps over a slab of n x n planes
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

// ---------------------------------------------------------------------------
// The kernel (v7 in DESIGN.md's history): one CTA per SM, 512 threads, a 64x32
// column tile streamed over i through a 3-stage TMA ring (c, u_b, u_1 halo
// boxes + the c_b / u_1_b tiles).  The shared-memory crossbar bounded the
// earlier single-role design (~160 B/pt incl. TMA fills); this one needs ~115:
//   * warps [0,8) carry Lap(u_1) (emit c_b), warps [8,16) the q stencil
//     (emit u_1_b); every thread owns 2 rows x 4 k-points of ONE field, so the
//     j-direction reads (2R+2 rows per 8 points instead of 4R+2) are shared
//     by the two rows in registers;
//   * g = 2 D c u_b [y in B] is produced inside the q-pass (the thread that
//     already holds c and u_b of that centre), so the centres are not re-read.
template <int R, int RING>
__device__ __forceinline__ void field2x4(const float* F, int r0, int col, float w0,
                                         const float (&wr)[R + 1], float4 (&acc)[RING][2],
                                         int ph) {
  constexpr int BW = 72;
  const float* row0 = F + r0 * BW + col;
  const float4 b0 = lds4(row0), b1 = lds4(row0 + BW);
  float4 in0 = kstencil2<R>(lds4(row0 - 4), b0, lds4(row0 + 4), w0, wr);
  float4 in1 = kstencil2<R>(lds4(row0 + BW - 4), b1, lds4(row0 + BW + 4), w0, wr);
  in0 = fmas4(wr[1], b1, in0);
  in1 = fmas4(wr[1], b0, in1);
#pragma unroll
  for (int t = -R; t <= R + 1; t++) {
    if (t == 0 || t == 1) continue;
    const float4 v = lds4(row0 + t * BW);
    const int d0 = t < 0 ? -t : t, d1 = t - 1 < 0 ? 1 - t : t - 1;
    if (d0 <= R) in0 = fmas4(wr[d0], v, in0);
    if (d1 <= R) in1 = fmas4(wr[d1], v, in1);
  }
  acc[ph][0] = add4(acc[ph][0], in0);
  acc[ph][1] = add4(acc[ph][1], in1);
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

template <int MODE>
struct StarTile7 {
  static constexpr int R = Star3<MODE>::R;
  static constexpr int TK = 64, TJ = 32, HK = 4, HJ = R;
  static constexpr int BW = TK + 2 * HK;
  static constexpr int BJ = TJ + 2 * HJ;
  static constexpr int RING = 2 * R + 1;
#ifndef SGB_V7_NQB
#define SGB_V7_NQB 2
#endif
#ifndef SGB_V7_QX
#define SGB_V7_QX 2
#endif
#ifndef SGB_V7_PF_TILES
#define SGB_V7_PF_TILES 1
#endif
  static constexpr int NS = 3, NQB = SGB_V7_NQB;
  static constexpr int ROLE = 16 * (TJ / 2);  // 256 threads per field
  static constexpr int THREADS = 2 * ROLE;
  static constexpr int BOX_BYTES = BW * BJ * 4;
  static constexpr int BF = ((BOX_BYTES + 127) / 128) * 128 / 4;
  static constexpr int TILE = TK * TJ;
  static constexpr int NT = Star3<MODE>::kU2 ? 3 : 2;
  static constexpr int SF = 3 * BF + NT * TILE;
  // g is written by q-pass threads and read by other (Lap) threads R planes
  // later, after one more barrier; a fast thread may already run the next
  // plane's q-pass, so the ring needs R + 2 slots (slot (it+1) != (it-R)).
  static constexpr int QD = R + SGB_V7_QX;
  static constexpr int QELEMS = (BW / 4) * BJ;
  static constexpr int EPT = (QELEMS + THREADS - 1) / THREADS;
  static constexpr size_t SMEM = (size_t)(NS * SF + NQB * BF + QD * TILE) * 4 + NS * 8;
  static_assert(RING % NS == 0, "static stage index");
};

// One non-blocking side stream (+ fork/join events) per device, created on
// first use; lets the frame kernel overlap the interior kernel.  Fork/join by
// events, so it is legal inside CUDA graph capture.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
inline SideStream* side_stream() {
  static SideStream per_dev[64];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  SideStream& ss = per_dev[dev];
  if (!ss.s) {
    if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
      ss.s = nullptr;
      return nullptr;
    }
  }
  return &ss;
}

// Tile map: interior tiles (halo box inside [lo, hi] in j and k) form the
// rectangle tk in [ik0, ik1) x tj in [ij0, ij1); the rest is a frame.  The
// INT=true instantiation runs the rectangle (k fastest) with no mask code at
// all, INT=false the frame; both are launched back to back.
struct TileMap {
  int tiles_k, tiles_j, ik0, ik1, ij0, ij1;
  __host__ __device__ int n_interior() const {
    return (ik1 > ik0 && ij1 > ij0) ? (ik1 - ik0) * (ij1 - ij0) : 0;
  }
  __host__ __device__ int n_frame() const { return tiles_k * tiles_j - n_interior(); }
  __device__ void interior(int t, int& tk, int& tj) const {
    const int w = ik1 - ik0;
    tk = ik0 + t % w;
    tj = ij0 + t / w;
  }
  __device__ void frame(int b, int& tk, int& tj) const {
    if (n_interior() == 0) {
      tk = b % tiles_k;
      tj = b / tiles_k;
      return;
    }
    const int top = ij0 * tiles_k;
    const int side = ik0 + (tiles_k - ik1);
    const int mid = (ij1 - ij0) * side;
    if (b < top) {
      tk = b % tiles_k;
      tj = b / tiles_k;
    } else if (b < top + mid) {
      const int m = b - top, r = m % side;
      tj = ij0 + m / side;
      tk = r < ik0 ? r : ik1 + (r - ik0);
    } else {
      const int m = b - top - mid;
      tk = m % tiles_k;
      tj = ij1 + m / tiles_k;
    }
  }
};

// Halo planes read straight from the neighbouring ranks' arrays (fused
// exchange: peer memory over NVLink via CUDA IPC, or any device-visible
// pointer): input planes below the local planes come from the lower
// neighbour's maps, above them from the upper neighbour's.
struct PeerHalo {
  CUtensorMap c[2], ub[2], u1[2];  // [0] lower neighbour, [1] upper neighbour
  int base[2];                     // global plane of the neighbour's array plane 0
  int has[2];
  int own0, own1;                  // planes held locally (global)
};

// One plane's TMA issue (elected thread): the c / u_b / u_1 halo boxes of
// input plane p -- from the neighbour's arrays when p lies outside the local
// planes and a PeerHalo is given -- and the c_b / u_1_b (/ u_2_b) tiles.  Kept
// out of line: it runs once per plane in one thread, and inlining it into
// every unrolled plane of both tile bodies costs instruction-cache misses.
__device__ __noinline__ void v7_issue(float* dst, uint64_t* bar, const CUtensorMap* tm_c,
                                      const CUtensorMap* tm_ub, const CUtensorMap* tm_u1,
                                      const CUtensorMap* tm_cb, const CUtensorMap* tm_u1b,
                                      const CUtensorMap* tm_u2b, const PeerHalo* peer, int p,
                                      int pl, int k0, int j0, int HK, int HJ, int ulo, int R,
                                      int BF, int TILE, int box_bytes, bool emit, bool u2,
                                      bool u1b) {
  tma::mbar_arrive_expect_tx(
      bar, 3 * box_bytes + ((emit ? (u1b ? 2 : 1) : 0) + (u2 ? 1 : 0)) * TILE * 4);
  const CUtensorMap *mc = tm_c, *mub = tm_ub, *mu1 = tm_u1;
  int pin = pl;
  if (peer) {  // uniform per plane: which array holds input plane p
    const int side = p < peer->own0 ? 0 : (p >= peer->own1 ? 1 : -1);
    if (side >= 0 && peer->has[side]) {
      mc = &peer->c[side];
      mub = &peer->ub[side];
      mu1 = &peer->u1[side];
      pin = p - peer->base[side];
    }
  }
  tma::load_3d(dst + 0 * BF, mc, bar, k0 - HK, j0 - HJ, pin);
  tma::load_3d(dst + 1 * BF, mub, bar, k0 - HK - ulo, j0 - HJ - ulo, pin);
  tma::load_3d(dst + 2 * BF, mu1, bar, k0 - HK, j0 - HJ, pin);
  if (emit) {
    tma::load_3d(dst + 3 * BF, tm_cb, bar, k0, j0, pl - R);
    if (u1b) tma::load_3d(dst + 3 * BF + TILE, tm_u1b, bar, k0, j0, pl - R);
  }
  if (u2) tma::load_3d(dst + 3 * BF + 2 * TILE, tm_u2b, bar, k0, j0, pl);
}

template <int MODE, bool INT, bool UBW>
__device__ __forceinline__ void star3_v7_body(
    const CUtensorMap& tm_c, const CUtensorMap& tm_ub, const CUtensorMap& tm_u1,
    const CUtensorMap& tm_cb, const CUtensorMap& tm_u1b, const CUtensorMap& tm_u2b,
    float* __restrict__ c_b, float* __restrict__ u_1_b, float* __restrict__ u_2_b, int n,
    int i_base, int lo, int hi, int out_i0, int out_i1, int chunk, int tk, int tj, float D,
    const PeerHalo* peer = nullptr, int PF = 0) {
  using Tl = StarTile7<MODE>;
  using S3 = Star3<MODE>;
  constexpr int R = Tl::R, HJ = Tl::HJ, HK = Tl::HK, BW = Tl::BW, TK = Tl::TK;
  constexpr int RING = Tl::RING, NS = Tl::NS, NQB = Tl::NQB, BF = Tl::BF, QD = Tl::QD;
  constexpr int SF = Tl::SF, TILE = Tl::TILE, ROLE = Tl::ROLE;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);  // [NS][c, ub, u1, cb, u1b, (u2b)]
  float* qbuf = stage + NS * SF;                       // [NQB][box]
  float* gq = qbuf + NQB * BF;                         // [QD][TJ][TK] (g of centres)
  uint64_t* bars = reinterpret_cast<uint64_t*>(gq + QD * TILE);

  const int tid = threadIdx.x;
  const bool q_role = tid >= ROLE;  // warp-uniform
  const int rt = q_role ? tid - ROLE : tid;
  const int tx = rt & 15, ty = rt >> 4;  // 4 k-points x rows 2ty, 2ty+1
  const int k0 = tk * TK, j0 = tj * Tl::TJ;
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
  const int ulo = UBW ? lo : 0;  // u_b map origin (windowed map: TMA does the mask)
  auto issue = [&](int it) {
    const int s = it % NS;
    float* dst = stage + s * SF;
    const int p = pstart + it;
    const int pl = p - i_base;
    const bool emit = it >= 2 * R;
    const bool u2 = S3::kU2 && p >= o_begin && p < o_end;
    if (peer) {  // fused-halo launches only (out of line: I-cache, see v7_issue)
      v7_issue(dst, &bars[s], &tm_c, &tm_ub, &tm_u1, &tm_cb, &tm_u1b, &tm_u2b, peer, p, pl, k0,
               j0, HK, HJ, ulo, R, BF, TILE, Tl::BOX_BYTES, emit, u2, !S3::kU1bFresh);
      return;
    }
    // fresh u_1_b (MODE 4): its old tile is not needed
    tma::mbar_arrive_expect_tx(
        &bars[s], 3 * Tl::BOX_BYTES +
                      ((emit ? (S3::kU1bFresh ? 1 : 2) : 0) + (u2 ? 1 : 0)) * TILE * 4);
    tma::load_3d(dst + 0 * BF, &tm_c, &bars[s], k0 - HK, j0 - HJ, pl);
    tma::load_3d(dst + 1 * BF, &tm_ub, &bars[s], k0 - HK - ulo, j0 - HJ - ulo, pl);
    tma::load_3d(dst + 2 * BF, &tm_u1, &bars[s], k0 - HK, j0 - HJ, pl);
    if (emit) {
      tma::load_3d(dst + 3 * BF, &tm_cb, &bars[s], k0, j0, pl - R);
      if (!S3::kU1bFresh) tma::load_3d(dst + 3 * BF + TILE, &tm_u1b, &bars[s], k0, j0, pl - R);
    }
    if (u2) tma::load_3d(dst + 3 * BF + 2 * TILE, &tm_u2b, &bars[s], k0, j0, pl);
    // L2 prefetch PF planes beyond the ring (the shared-memory ring holds
    // NS planes; a plane's boxes then arrive from L2, not DRAM)
    if (PF > 0 && it + PF < P) {
      const int q = pl + PF;
      tma::prefetch_3d(&tm_c, k0 - HK, j0 - HJ, q);
      tma::prefetch_3d(&tm_ub, k0 - HK - ulo, j0 - HJ - ulo, q);
      tma::prefetch_3d(&tm_u1, k0 - HK, j0 - HJ, q);
      if (SGB_V7_PF_TILES && it + PF >= 2 * R) {
        tma::prefetch_3d(&tm_cb, k0, j0, q - R);
        if (!S3::kU1bFresh) tma::prefetch_3d(&tm_u1b, k0, j0, q - R);
      }
    }
  };
  if (tid == 0)
    for (int it = 0; it < NS && it < P; it++) issue(it);

  const int jr0 = j0 + 2 * ty, kc = k0 + 4 * tx;
  const int r0 = 2 * ty + HJ, col = HK + 4 * tx;
  const int trow = 2 * ty * TK + 4 * tx;  // offset of row 2ty in a 64x32 tile
  const long long plane = (long long)n * n;
  const int coff = jr0 * n + kc;  // in-plane offset (n*n < 2^31)

  // q-pass elements of this thread (fixed for all planes): smem offset in the
  // box and, for centre elements, offset of its g in the 64x32 g tile
  int qoff[Tl::EPT], goff[Tl::EPT];
#pragma unroll
  for (int m = 0; m < Tl::EPT; m++) {
    const int e = tid + m * Tl::THREADS;
    const int row = e / (BW / 4), c4 = e - row * (BW / 4);
    qoff[m] = e < Tl::QELEMS ? row * BW + 4 * c4 : -1;
    goff[m] = (e < Tl::QELEMS && row >= HJ && row < HJ + Tl::TJ && c4 >= 1 && c4 <= TK / 4)
                  ? (row - HJ) * TK + 4 * (c4 - 1)
                  : -1;
  }
  // Frame tiles: every (j, k) predicate is plane-independent, so it is
  // evaluated once here into bit masks (only the i terms vary per plane).
  //   qmask bit 4m+x : u_b element x of q-pass element m inside [lo, hi]^2
  //   fm bits 0-7   : centre (h, x) with j, k in [lo, hi]          (set A)
  //   fm bits 8-15  : centre (h, x) one coordinate out by <= R     (set B)
  //   fm bits 16-19 : k = kc + x in [lo, hi]
  //   fm bits 20-21 : row h in [lo, hi] and inside the grid
  //   fm bits 22-23 : row h inside the grid
  uint32_t qmask = 0, fm = 0;
  if (!INT) {
#pragma unroll
    for (int m = 0; m < Tl::EPT; m++) {
      if (qoff[m] < 0 || UBW) continue;
      const int row = qoff[m] / BW, c4 = (qoff[m] - row * BW) >> 2;
      const int jg = j0 - HJ + row, kg = k0 - HK + 4 * c4;
      const bool rm = jg >= lo && jg <= hi;
#pragma unroll
      for (int x = 0; x < 4; x++)
        if (rm && kg + x >= lo && kg + x <= hi) qmask |= 1u << (4 * m + x);
    }
#pragma unroll
    for (int x = 0; x < 4; x++)
      if (kc + x >= lo && kc + x <= hi) fm |= 1u << (16 + x);
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int j = jr0 + h;
      const bool grid = j < n && kc < n;
      const bool jin = j >= lo && j <= hi;
      const int jout = j < lo ? lo - j : (j > hi ? j - hi : 0);
      if (grid) fm |= 1u << (22 + h);
      if (grid && jin) fm |= 1u << (20 + h);
#pragma unroll
      for (int x = 0; x < 4; x++) {
        const int k = kc + x;
        const int kout = k < lo ? lo - k : (k > hi ? k - hi : 0);
        if (jout == 0 && kout == 0) fm |= 1u << (4 * h + x);
        if ((jout > 0) + (kout > 0) == 1 && jout <= R && kout <= R) fm |= 1u << (8 + 4 * h + x);
      }
    }
  }

  float4 acc[RING][2];
#pragma unroll
  for (int s = 0; s < RING; s++) acc[s][0] = acc[s][1] = make_float4(0.f, 0.f, 0.f, 0.f);

  for (int base = 0; base < P; base += RING) {
    const int par0 = base / NS;
#pragma unroll
    for (int ph = 0; ph < RING; ph++) {
      const int it = base + ph;
      if (it < P) {
        const int s = ph % NS;
        const int p = pstart + it;
        const float* Cs = stage + s * SF;
        const float* UBs = Cs + BF;
        const float* U1s = Cs + 2 * BF;
        float* Q = qbuf + ((it & 1) ? BF : 0);
        float* G = gq + (it % QD) * TILE;
        const bool emit = it >= 2 * R;
        const int o = p - R;
        const bool pin = p >= lo && p <= hi;
        const bool oin = o >= lo && o <= hi;

        tma::mbar_wait(&bars[s], (par0 + ph / NS) & 1);
        float4 old[2];
        {
          const float* OLD = Cs + 3 * BF + (q_role ? TILE : 0) + trow;
          if (S3::kU1bFresh && q_role) {  // u_1_b starts from zero this step
            old[0] = old[1] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            old[0] = lds4(OLD);
            old[1] = lds4(OLD + TK);
          }
        }

        // ---- q over the halo box; g for the centre elements
#pragma unroll
        for (int m = 0; m < Tl::EPT; m++) {
          if (qoff[m] >= 0) {
            const int qo = qoff[m];
            const bool centre = goff[m] >= 0;
            float4 qv = make_float4(0.f, 0.f, 0.f, 0.f), gv = qv;
            if (pin) {
              const float4 cv = lds4(Cs + qo);
              float4 uv = lds4(UBs + qo);
              if (!INT && !UBW) {
                const uint32_t mk = qmask >> (4 * m);
                uv = make_float4(mk & 1 ? uv.x : 0.f, mk & 2 ? uv.y : 0.f, mk & 4 ? uv.z : 0.f,
                                 mk & 8 ? uv.w : 0.f);
              }
              const float4 du = muls4(D, uv);
              qv = mul4(S3::kC2 ? mul4(cv, cv) : cv, du);
              if (centre) gv = S3::kC2 ? mul4(muls4(2.f, cv), du) : du;
            }
            *reinterpret_cast<float4*>(Q + qo) = qv;
            if (centre) *reinterpret_cast<float4*>(G + goff[m]) = gv;
          }
        }
        // ---- q role: 2 u_b centre term (and u_2_b at plane p)
        if (q_role && pin) {
          float* u2_plane = u_2_b + (long long)(p - i_base) * plane;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            float4 ubm = lds4(UBs + (r0 + h) * BW + col);
            bool kin[4] = {true, true, true, true}, jin = true;
            if (!INT) {
              const uint32_t mk = fm >> (4 * h);
              jin = (fm >> (20 + h)) & 1;
#pragma unroll
              for (int x = 0; x < 4; x++) kin[x] = (fm >> (16 + x)) & 1;
              if (!UBW)
                ubm = make_float4(mk & 1 ? ubm.x : 0.f, mk & 2 ? ubm.y : 0.f, mk & 4 ? ubm.z : 0.f,
                                mk & 8 ? ubm.w : 0.f);
            }
            acc[ph][h] = fmas4(2.f, ubm, acc[ph][h]);
            if (S3::kU2 && jin && p >= o_begin &&
                p < o_end) {
              const float4 u2 = lds4(Cs + 3 * BF + 2 * TILE + trow + h * TK);
              __stcs(reinterpret_cast<float4*>(u2_plane + coff + h * n),
                     make_float4(kin[0] ? u2.x - ubm.x : u2.x, kin[1] ? u2.y - ubm.y : u2.y,
                                 kin[2] ? u2.z - ubm.z : u2.z, kin[3] ? u2.w - ubm.w : u2.w));
            }
          }
        }
        // ---- time-loop u_2 partial (MODE 3): u_2_b[p] = -u_b[p] on B, 0
        // elsewhere, for every owned plane p of this chunk (sgb_box_set's
        // values bit for bit: 0 - u is 0 + (-1) u for every u)
        if (S3::kU2Set && q_role && p >= o_begin && p < o_end) {
          float* u2_plane = u_2_b + (long long)(p - i_base) * plane;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            if (!INT && !((fm >> (22 + h)) & 1)) continue;  // row outside the grid
            float4 ubm = lds4(UBs + (r0 + h) * BW + col);
            bool m[4] = {pin, pin, pin, pin};
            if (!INT) {
              const bool jin = (fm >> (20 + h)) & 1;
#pragma unroll
              for (int x = 0; x < 4; x++) m[x] = pin && jin && ((fm >> (16 + x)) & 1);
            }
            __stcs(reinterpret_cast<float4*>(u2_plane + coff + h * n),
                   make_float4(m[0] ? 0.f - ubm.x : 0.f, m[1] ? 0.f - ubm.y : 0.f,
                               m[2] ? 0.f - ubm.z : 0.f, m[3] ? 0.f - ubm.w : 0.f));
          }
        }
        __syncthreads();
        if (tid == 0 && it >= 1 && it - 1 + NS < P) issue(it - 1 + NS);

        field2x4<R, RING>(q_role ? Q : U1s, r0, col, w0, wr, acc, ph);

        // ---- emit output plane o = p - R
        if (emit) {
          const int es = (ph + R + 1) % RING;
          const long long obase = (long long)(o - i_base) * plane;
          if (!q_role) {
            if (oin) {
              const float* Go = gq + ((it - R) % QD) * TILE + trow;
              float* cb_plane = c_b + obase;
#pragma unroll
              for (int h = 0; h < 2; h++) {
                float4 nv = fma4(lds4(Go + h * TK), acc[es][h], old[h]);
                if (!INT) {
                  if (!((fm >> (20 + h)) & 1)) continue;
                  const uint32_t mk = fm >> 16;
                  nv = make_float4(mk & 1 ? nv.x : old[h].x, mk & 2 ? nv.y : old[h].y,
                                   mk & 4 ? nv.z : old[h].z, mk & 8 ? nv.w : old[h].w);
                }
                __stcs(reinterpret_cast<float4*>(cb_plane + coff + h * n), nv);
              }
            }
          } else {
            const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
            float* u1b_plane = u_1_b + obase;
            if (INT) {
              if (oout <= R) {
#pragma unroll
                for (int h = 0; h < 2; h++)
                  __stcs(reinterpret_cast<float4*>(u1b_plane + coff + h * n),
                         add4(old[h], acc[es][h]));
              } else if (S3::kU1bFresh) {  // not reached: zero
#pragma unroll
                for (int h = 0; h < 2; h++)
                  __stcs(reinterpret_cast<float4*>(u1b_plane + coff + h * n),
                         make_float4(0.f, 0.f, 0.f, 0.f));
              }
            } else {
              // reached iff at most one coordinate is outside [lo, hi], by <= R
              const uint32_t reach =
                  oout == 0 ? (fm | (fm >> 8)) & 0xff : (oout <= R ? fm & 0xff : 0u);
#pragma unroll
              for (int h = 0; h < 2; h++) {
                const uint32_t mk = reach >> (4 * h);
                if (!((fm >> (22 + h)) & 1) || (!S3::kU1bFresh && !(mk & 0xf))) continue;
                const float4 a = acc[es][h];
                const float4 nv = make_float4(mk & 1 ? old[h].x + a.x : old[h].x,
                                              mk & 2 ? old[h].y + a.y : old[h].y,
                                              mk & 4 ? old[h].z + a.z : old[h].z,
                                              mk & 8 ? old[h].w + a.w : old[h].w);
                __stcs(reinterpret_cast<float4*>(u1b_plane + coff + h * n), nv);
              }
            }
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// v8 (interior tiles of the radius-4 specs MODE 2 / 4; bitwise = v7):
// the v7 tile, ring and shared-memory layout with HALF the threads -- 256,
// each owning 4 rows x 4 k points of one field -- so the per-plane work that
// does not scale with points (barrier, mbarrier wait, bookkeeping, the j rows
// shared by a thread's rows: 12 row loads per 4 rows instead of 10 per 2)
// is spread over twice the points, at 8 warps per SM and 222 registers.
template <int MODE>
struct StarTile8 : StarTile7<MODE> {
  static constexpr int ROLE = 16 * (StarTile7<MODE>::TJ / 4);  // 128 threads per field
  static constexpr int THREADS = 2 * ROLE;
  static constexpr int EPT = (StarTile7<MODE>::QELEMS + THREADS - 1) / THREADS;
  // two mbarriers per stage: A (c, u_b boxes: dead after the q pass) and B
  // (u_1 box, output tiles)
  static constexpr size_t SMEM = StarTile7<MODE>::SMEM + StarTile7<MODE>::NS * 8;
};

template <int R, int RING>
__device__ __forceinline__ void field4x4(const float* F, int r0, int col, float w0,
                                         const float (&wr)[R + 1], float4 (&acc)[RING][4],
                                         int ph) {
  constexpr int BW = 72;
  const float* row0 = F + r0 * BW + col;
  float4 b[4], in[4];
#pragma unroll
  for (int h = 0; h < 4; h++) {
    b[h] = lds4(row0 + h * BW);
    in[h] = kstencil2<R>(lds4(row0 + h * BW - 4), b[h], lds4(row0 + h * BW + 4), w0, wr);
  }
  // j direction, each row's terms in EXACTLY field2x4's order (its pair
  // partner first, then the other rows bottom to top), so v8 and v7 give the
  // same bits: rows of the 4-row group from registers, the rest from shared
  // memory (the compiler merges the repeated loads)
#pragma unroll
  for (int pos = 0; pos < 2 * R; pos++) {
#pragma unroll
    for (int h = 0; h < 4; h++) {
      // offsets of row h relative to itself, in v7's order for its pair slot
      int off;
      if ((h & 1) == 0) off = pos == 0 ? 1 : (pos <= R ? pos - 1 - R : pos - R + 1);
      else off = pos == 0 ? -1 : (pos < R ? pos - 1 - R : pos - R + 1);
      const int t = h + off;
      const int d = off < 0 ? -off : off;
      const float4 v = (t >= 0 && t <= 3) ? b[t < 0 ? 0 : (t > 3 ? 3 : t)] : lds4(row0 + t * BW);
      in[h] = fmas4(wr[d], v, in[h]);
    }
  }
  // i direction: this plane's sum into its slot, its centre values into the
  // neighbouring planes' slots (the v7 ring)
#pragma unroll
  for (int h = 0; h < 4; h++) {
    acc[ph][h] = add4(acc[ph][h], in[h]);
    acc[(ph + R) % RING][h] = muls4(wr[R], b[h]);
#pragma unroll
    for (int r = 1; r <= R; r++) {
      if (r < R) acc[(ph + r) % RING][h] = fmas4(wr[r], b[h], acc[(ph + r) % RING][h]);
      acc[(ph + RING - r) % RING][h] = fmas4(wr[r], b[h], acc[(ph + RING - r) % RING][h]);
    }
  }
}

template <int MODE, bool INT>
__device__ __forceinline__ void star3_v8_body(
    const CUtensorMap& tm_c, const CUtensorMap& tm_ub, const CUtensorMap& tm_u1,
    const CUtensorMap& tm_cb, const CUtensorMap& tm_u1b, float* __restrict__ c_b,
    float* __restrict__ u_1_b, int n, int i_base, int lo, int hi, int out_i0, int out_i1,
    int chunk, int tk, int tj, float D, int ob = -1, int oe = -1, bool again = false) {
  // ob / oe: an explicit output plane range (else chunk blockIdx.y of
  // [out_i0, out_i1)); again: the CTA ran a range before -- its mbarriers are
  // invalidated and set up anew (every load it issued was consumed)
  using Tl = StarTile8<MODE>;
  using S3 = Star3<MODE>;
  static_assert(!S3::kU2 && !S3::kU2Set, "v8: radius-4 specs without u_2 partials");
  constexpr int R = Tl::R, HJ = Tl::HJ, HK = Tl::HK, BW = Tl::BW, TK = Tl::TK;
  constexpr int RING = Tl::RING, NS = Tl::NS, BF = Tl::BF, QD = Tl::QD;
  constexpr int SF = Tl::SF, TILE = Tl::TILE, ROLE = Tl::ROLE;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);
  float* qbuf = stage + NS * SF;
  float* gq = qbuf + Tl::NQB * BF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(gq + QD * TILE);

  const int tid = threadIdx.x;
  const bool q_role = tid >= ROLE;
  const int rt = q_role ? tid - ROLE : tid;
  const int tx = rt & 15, ty = rt >> 4;  // 4 k-points x rows 4ty .. 4ty+3
  const int k0 = tk * TK, j0 = tj * Tl::TJ;
  const int o_begin = ob >= 0 ? ob : out_i0 + blockIdx.y * chunk;
  const int o_end = ob >= 0 ? oe : min(o_begin + chunk, out_i1);
  if (o_begin >= o_end) return;
  const int pstart = o_begin - R;
  const int P = (o_end - o_begin) + 2 * R;

  const float w0 = S3::template w<float>(0);
  float wr[R + 1];
  wr[0] = w0;
#pragma unroll
  for (int r = 1; r <= R; r++) wr[r] = S3::template w<float>(r);

  uint64_t* barsB = bars + NS;
  if (again) __syncthreads();  // every thread is done with the previous range
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < 2 * NS; s++) {
      if (again) tma::mbar_inval(&bars[s]);
      tma::mbar_init(&bars[s], 1);
    }
    tma::fence_barrier_init();
  }
  __syncthreads();
  // A half of a stage: the c / u_b boxes, read only by the q pass (before the
  // plane's barrier), so plane it + NS is requested right after plane it's
  // barrier -- one plane earlier than the B half (u_1 box, output tiles),
  // which is read after the barrier and freed at the next one
  auto issueA = [&](int it) {
    const int s = it % NS;
    float* dst = stage + s * SF;
    const int pl = pstart + it - i_base;
    tma::mbar_arrive_expect_tx(&bars[s], 2 * Tl::BOX_BYTES);
    tma::load_3d(dst + 0 * BF, &tm_c, &bars[s], k0 - HK, j0 - HJ, pl);
    tma::load_3d(dst + 1 * BF, &tm_ub, &bars[s], k0 - HK - lo, j0 - HJ - lo, pl);
  };
  auto issueB = [&](int it) {
    const int s = it % NS;
    float* dst = stage + s * SF;
    const int pl = pstart + it - i_base;
    const bool emit = it >= 2 * R;
    tma::mbar_arrive_expect_tx(
        &barsB[s], Tl::BOX_BYTES + (emit ? (S3::kU1bFresh ? 1 : 2) : 0) * TILE * 4);
    tma::load_3d(dst + 2 * BF, &tm_u1, &barsB[s], k0 - HK, j0 - HJ, pl);
    if (emit) {
      tma::load_3d(dst + 3 * BF, &tm_cb, &barsB[s], k0, j0, pl - R);
      if (!S3::kU1bFresh) tma::load_3d(dst + 3 * BF + TILE, &tm_u1b, &barsB[s], k0, j0, pl - R);
    }
  };
  if (tid == 0)
    for (int it = 0; it < NS && it < P; it++) {
      issueA(it);
      issueB(it);
    }

  const int jr0 = j0 + 4 * ty, kc = k0 + 4 * tx;
  const int r0 = 4 * ty + HJ, col = HK + 4 * tx;
  const int trow = 4 * ty * TK + 4 * tx;
  const long long plane = (long long)n * n;
  const int coff = jr0 * n + kc;

  int qoff[Tl::EPT], goff[Tl::EPT];
#pragma unroll
  for (int m = 0; m < Tl::EPT; m++) {
    const int e = tid + m * Tl::THREADS;
    const int row = e / (BW / 4), c4 = e - row * (BW / 4);
    qoff[m] = e < Tl::QELEMS ? row * BW + 4 * c4 : -1;
    goff[m] = (e < Tl::QELEMS && row >= HJ && row < HJ + Tl::TJ && c4 >= 1 && c4 <= TK / 4)
                  ? (row - HJ) * TK + 4 * (c4 - 1)
                  : -1;
  }

  // frame tiles: plane-independent per-point masks (v7's, for 4 rows):
  //   fmA bit 4h+x: centre (h, x) with j, k in [lo, hi]
  //   fmB bit 4h+x: exactly one of j, k outside [lo, hi], by <= R
  //   fk  bit x: k = kc + x in [lo, hi]; fr bit h: row h in [lo, hi] and in
  //   the grid; fg bit h: row h in the grid (kc < n: n % 4 == 0 on this path)
  uint32_t fmA = 0, fmB = 0, fk = 0, fr = 0, fg = 0;
  if (!INT) {
#pragma unroll
    for (int x = 0; x < 4; x++)
      if (kc + x >= lo && kc + x <= hi) fk |= 1u << x;
#pragma unroll
    for (int h = 0; h < 4; h++) {
      const int j = jr0 + h;
      const bool grid = j < n && kc < n;
      const int jout = j < lo ? lo - j : (j > hi ? j - hi : 0);
      if (grid) fg |= 1u << h;
      if (grid && jout == 0) fr |= 1u << h;
#pragma unroll
      for (int x = 0; x < 4; x++) {
        const int k = kc + x;
        const int kout = k < lo ? lo - k : (k > hi ? k - hi : 0);
        if (jout == 0 && kout == 0) fmA |= 1u << (4 * h + x);
        if ((jout > 0) + (kout > 0) == 1 && jout <= R && kout <= R) fmB |= 1u << (4 * h + x);
      }
    }
  }

  float4 acc[RING][4];
#pragma unroll
  for (int s = 0; s < RING; s++)
#pragma unroll
    for (int h = 0; h < 4; h++) acc[s][h] = make_float4(0.f, 0.f, 0.f, 0.f);

  for (int base = 0; base < P; base += RING) {
    const int par0 = base / NS;
#pragma unroll
    for (int ph = 0; ph < RING; ph++) {
      const int it = base + ph;
      if (it < P) {
        const int s = ph % NS;
        const int p = pstart + it;
        const float* Cs = stage + s * SF;
        const float* UBs = Cs + BF;
        const float* U1s = Cs + 2 * BF;
        float* Q = qbuf + ((it & 1) ? BF : 0);
        float* G = gq + (it % QD) * TILE;
        const bool emit = it >= 2 * R;
        const int o = p - R;
        const bool pin = p >= lo && p <= hi;

        const uint32_t par = (par0 + ph / NS) & 1;
        tma::mbar_wait(&bars[s], par);
#pragma unroll
        for (int m = 0; m < Tl::EPT; m++) {
          if (qoff[m] >= 0) {
            const int qo = qoff[m];
            const bool centre = goff[m] >= 0;
            float4 qv = make_float4(0.f, 0.f, 0.f, 0.f), gv = qv;
            if (pin) {
              const float4 cv = lds4(Cs + qo);
              const float4 du = muls4(D, lds4(UBs + qo));
              qv = mul4(mul4(cv, cv), du);
              if (centre) gv = mul4(muls4(2.f, cv), du);
            }
            *reinterpret_cast<float4*>(Q + qo) = qv;
            if (centre) *reinterpret_cast<float4*>(G + goff[m]) = gv;
          }
        }
        if (q_role && pin) {
#pragma unroll
          for (int h = 0; h < 4; h++)
            acc[ph][h] = fmas4(2.f, lds4(UBs + (r0 + h) * BW + col), acc[ph][h]);
        }
        __syncthreads();
        if (tid == 0) {  // in the order they are needed: B of plane it+NS-1 first
          if (it >= 1 && it - 1 + NS < P) issueB(it - 1 + NS);
          // the early A half pays for the fresh form only: with the second
          // output tile (accumulating form) in the late half it loses 9-11 %,
          // so there both halves of a plane are requested together
          if (S3::kU1bFresh) {
            if (it + NS < P) issueA(it + NS);
          } else if (it >= 1 && it - 1 + NS < P) {
            issueA(it - 1 + NS);
          }
        }
        tma::mbar_wait(&barsB[s], par);

        field4x4<R, RING>(q_role ? Q : U1s, r0, col, w0, wr, acc, ph);

        if (emit) {
          const int es = (ph + R + 1) % RING;
          float* obase = (q_role ? u_1_b : c_b) + (long long)(o - i_base) * plane + coff;
          const float* OLD = Cs + 3 * BF + (q_role ? TILE : 0) + trow;
          if (!q_role) {
            if (o >= lo && o <= hi) {
              const float* Go = gq + ((it - R) % QD) * TILE + trow;
#pragma unroll
              for (int h = 0; h < 4; h++) {
                const float4 old = lds4(OLD + h * TK);
                float4 nv = fma4(lds4(Go + h * TK), acc[es][h], old);
                if (!INT) {
                  if (!((fr >> h) & 1)) continue;
                  nv = make_float4(fk & 1 ? nv.x : old.x, fk & 2 ? nv.y : old.y,
                                   fk & 4 ? nv.z : old.z, fk & 8 ? nv.w : old.w);
                }
                __stcs(reinterpret_cast<float4*>(obase + h * n), nv);
              }
            }
          } else if (!INT) {
            // reached iff at most one coordinate is outside [lo, hi], by <= R
            const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
            const uint32_t reach = oout == 0 ? (fmA | fmB) : (oout <= R ? fmA : 0u);
#pragma unroll
            for (int h = 0; h < 4; h++) {
              const uint32_t mk = (reach >> (4 * h)) & 0xf;
              if (!((fg >> h) & 1) || (!S3::kU1bFresh && !mk)) continue;
              const float4 old =
                  S3::kU1bFresh ? make_float4(0.f, 0.f, 0.f, 0.f) : lds4(OLD + h * TK);
              const float4 a = acc[es][h];
              __stcs(reinterpret_cast<float4*>(obase + h * n),
                     make_float4(mk & 1 ? old.x + a.x : old.x, mk & 2 ? old.y + a.y : old.y,
                                 mk & 4 ? old.z + a.z : old.z, mk & 8 ? old.w + a.w : old.w));
            }
          } else {
            const int oout = o < lo ? lo - o : (o > hi ? o - hi : 0);
            if (oout <= R) {
#pragma unroll
              for (int h = 0; h < 4; h++) {
                const float4 old =
                    S3::kU1bFresh ? make_float4(0.f, 0.f, 0.f, 0.f) : lds4(OLD + h * TK);
                __stcs(reinterpret_cast<float4*>(obase + h * n), add4(old, acc[es][h]));
              }
            } else if (S3::kU1bFresh) {
#pragma unroll
              for (int h = 0; h < 4; h++)
                __stcs(reinterpret_cast<float4*>(obase + h * n), make_float4(0.f, 0.f, 0.f, 0.f));
            }
          }
        }
      }
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(StarTile8<MODE>::THREADS, 1)
    star3_v8_kernel(const __grid_constant__ CUtensorMap tm_c,
                    const __grid_constant__ CUtensorMap tm_ub,
                    const __grid_constant__ CUtensorMap tm_u1,
                    const __grid_constant__ CUtensorMap tm_cb,
                    const __grid_constant__ CUtensorMap tm_u1b, float* __restrict__ c_b,
                    float* __restrict__ u_1_b, int n, int i_base, int lo, int hi, int out_i0,
                    int out_i1, int chunk, TileMap tmap, float D, int which) {
  // which: 0 interior rectangle, 1 frame (a single launch over all tiles
  // with a per-CTA body choice measured 1.75x slower: 8.1 vs 4.6 ms at 1024^3)
  int tk, tj;
  const bool interior = which == 0;
  if (interior)
    tmap.interior(blockIdx.x, tk, tj);
  else
    tmap.frame(blockIdx.x, tk, tj);
  if (interior)
    star3_v8_body<MODE, true>(tm_c, tm_ub, tm_u1, tm_cb, tm_u1b, c_b, u_1_b, n, i_base, lo, hi,
                              out_i0, out_i1, chunk, tk, tj, D);
  else
    star3_v8_body<MODE, false>(tm_c, tm_ub, tm_u1, tm_cb, tm_u1b, c_b, u_1_b, n, i_base, lo,
                               hi, out_i0, out_i1, chunk, tk, tj, D);
}

// Interior launch with a balanced last wave (v8, one chunk per column).  With
// T interior tiles on S SMs the last of ceil(T / S) waves runs T % S CTAs and
// leaves the other SMs idle for a whole column (1024^3: 420 tiles, 2.84
// waves).  Here the first `full` tiles run whole columns; of the remaining
// `rem` tiles the planes [out_i0, split) go to one CTA each and the planes
// [split, out_i1) of ALL of them to the gridDim.x - full - rem filler CTAs,
// filler f taking tiles full + f, full + f + nfill, ... -- so the fillers move
// through adjacent tiles in lock-step (halo rows shared in L2) and every SM
// finishes at about the same time.  Same arithmetic per point: bitwise equal.
template <int MODE>
__global__ void __launch_bounds__(StarTile8<MODE>::THREADS, 1)
    star3_v8_balanced(const __grid_constant__ CUtensorMap tm_c,
                      const __grid_constant__ CUtensorMap tm_ub,
                      const __grid_constant__ CUtensorMap tm_u1,
                      const __grid_constant__ CUtensorMap tm_cb,
                      const __grid_constant__ CUtensorMap tm_u1b, float* __restrict__ c_b,
                      float* __restrict__ u_1_b, int n, int i_base, int lo, int hi, int out_i0,
                      int out_i1, TileMap tmap, float D, int full, int rem, int split) {
  // one call site for the body (two inlined copies of its ~5 K instructions
  // thrash the instruction cache: 15 % slower)
  const int b = blockIdx.x;
  const bool filler = b >= full + rem;
  const int nfill = (int)gridDim.x - full - rem;
  const int t0 = filler ? full + (b - full - rem) : b;
  const int tend = filler ? full + rem : b + 1;
  const int step = filler ? nfill : 1;
  const int ob = filler ? split : out_i0;
  const int oe = (filler || b < full) ? out_i1 : split;
  bool again = false;
  for (int t = t0; t < tend; t += step) {
    int tk, tj;
    tmap.interior(t, tk, tj);
    star3_v8_body<MODE, true>(tm_c, tm_ub, tm_u1, tm_cb, tm_u1b, c_b, u_1_b, n, i_base, lo, hi,
                              out_i0, out_i1, 0, tk, tj, D, ob, oe, again);
    again = true;
  }
}

#define SGB_V7_PARAMS                                                                   \
  const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_ub,     \
      const __grid_constant__ CUtensorMap tm_u1, const __grid_constant__ CUtensorMap tm_cb, \
      const __grid_constant__ CUtensorMap tm_u1b,                                          \
      const __grid_constant__ CUtensorMap tm_u2b, float *__restrict__ c_b,                 \
      float *__restrict__ u_1_b, float *__restrict__ u_2_b, int n, int i_base, int lo,     \
      int hi, int out_i0, int out_i1, int chunk, TileMap tm, float D, int pf
#define SGB_V7_ARGS                                                                    \
  tm_c, tm_ub, tm_u1, tm_cb, tm_u1b, tm_u2b, c_b, u_1_b, u_2_b, n, i_base, lo, hi, out_i0, \
      out_i1, chunk

// INT=true runs the interior rectangle, INT=false the frame; UBW: u_b map is
// windowed to [lo, hi]^2 (TMA zero fill replaces the seed mask).
template <int MODE, bool INT, bool UBW>
__global__ void __launch_bounds__(StarTile7<MODE>::THREADS, 1) star3_v7_kernel(SGB_V7_PARAMS) {
  int tk, tj;
  if (INT)
    tm.interior(blockIdx.x, tk, tj);
  else
    tm.frame(blockIdx.x, tk, tj);
  star3_v7_body<MODE, INT, UBW>(SGB_V7_ARGS, tk, tj, D, nullptr, pf);
}

// One launch over all tiles in row-major order, each CTA running the body
// specialised for its tile, so frame and interior neighbours stream the same
// planes concurrently and share halo rows in L2.  Used for partial plane
// ranges (z-slabs, edge bands); for the full grid it is 1.2% faster at full
// clock but 1.5% slower in the sustained (power-capped) 200-step run
// bench.py measures, so the full grid keeps the split launch.
template <int MODE, bool UBW>
__global__ void __launch_bounds__(StarTile7<MODE>::THREADS, 1) star3_v7_unified(SGB_V7_PARAMS) {
  const int tk = blockIdx.x % tm.tiles_k, tj = blockIdx.x / tm.tiles_k;
  if (tk >= tm.ik0 && tk < tm.ik1 && tj >= tm.ij0 && tj < tm.ij1)
    star3_v7_body<MODE, true, UBW>(SGB_V7_ARGS, tk, tj, D, nullptr, pf);
  else
    star3_v7_body<MODE, false, UBW>(SGB_V7_ARGS, tk, tj, D, nullptr, pf);
}

// The same, with the halo planes read from the neighbours' arrays.
template <int MODE, bool UBW>
__global__ void __launch_bounds__(StarTile7<MODE>::THREADS, 1)
    star3_v7_unified_peer(SGB_V7_PARAMS, const __grid_constant__ PeerHalo peer) {
  const int tk = blockIdx.x % tm.tiles_k, tj = blockIdx.x / tm.tiles_k;
  if (tk >= tm.ik0 && tk < tm.ik1 && tj >= tm.ij0 && tj < tm.ij1)
    star3_v7_body<MODE, true, UBW>(SGB_V7_ARGS, tk, tj, D, &peer, pf);
  else
    star3_v7_body<MODE, false, UBW>(SGB_V7_ARGS, tk, tj, D, &peer, pf);
}

template <int MODE>
inline int star3_v7_gather(const Slab3& g, long long lo, long long hi, long long out_i0,
                           long long out_i1, float D, const float* c, float* c_b,
                           const float* u_1, float* u_1_b, float* u_2_b, const float* u_b,
                           cudaStream_t s, const char* name, const PeerHalo* peer = nullptr) {
  using Tl = StarTile7<MODE>;
  CUtensorMap maps[6];
  int rc = 0;
  rc |= encode_3d(&maps[0], c, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  int ubwin = 0;
  if (!opt_flag(OPT_NO_UBWIN)) {
    const int w = encode_3d_window(&maps[1], u_b, g.n, g.nplanes, lo, hi - lo + 1, Tl::BW, Tl::BJ,
                                   name);
    if (w < 0) return w;
    ubwin = w == 0;
  }
  if (!ubwin) rc |= encode_3d(&maps[1], u_b, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  rc |= encode_3d(&maps[2], u_1, g.n, g.nplanes, Tl::BW, Tl::BJ, name);
  rc |= encode_3d(&maps[3], c_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  rc |= encode_3d(&maps[4], u_1_b, g.n, g.nplanes, Tl::TK, Tl::TJ, name);
  rc |= encode_3d(&maps[5], Star3<MODE>::kU2 ? u_2_b : u_1_b, g.n, g.nplanes, Tl::TK, Tl::TJ,
                  name);
  if (rc) return SGB_EINVAL;
  {
    const void* ks[] = {(const void*)star3_v7_kernel<MODE, true, true>,
                        (const void*)star3_v7_kernel<MODE, true, false>,
                        (const void*)star3_v7_kernel<MODE, false, true>,
                        (const void*)star3_v7_kernel<MODE, false, false>,
                        (const void*)star3_v7_unified<MODE, true>,
                        (const void*)star3_v7_unified_peer<MODE, true>};
    for (const void* k : ks)
      if (int r = ensure_smem(k, Tl::SMEM, name)) return r;
  }
  TileMap tm;
  tm.tiles_k = (int)((g.n + Tl::TK - 1) / Tl::TK);
  tm.tiles_j = (int)((g.n + Tl::TJ - 1) / Tl::TJ);
  // interior: the whole halo box inside [lo, hi] (and inside the grid)
  auto first_in = [&](int T, int H) {  // smallest tile index t with t*T - H >= lo
    long long t = (lo + H + T - 1) / T;
    return (int)t;
  };
  auto end_in = [&](int T, int H, int tiles) {  // one past the last t with t*T+T+H-1 <= hi
    long long t = (hi - H + 1) / T;             // t*T + T + H - 1 <= hi  <=> t <= (hi-H+1)/T - 1
    return (int)std::min<long long>(t, tiles);
  };
  tm.ik0 = first_in(Tl::TK, Tl::HK);
  tm.ik1 = end_in(Tl::TK, Tl::HK, tm.tiles_k);
  tm.ij0 = first_in(Tl::TJ, Tl::HJ);
  tm.ij1 = end_in(Tl::TJ, Tl::HJ, tm.tiles_j);
  if (tm.ik1 <= tm.ik0 || tm.ij1 <= tm.ij0) tm.ik0 = tm.ik1 = tm.ij0 = tm.ij1 = 0;
  const long long nout = out_i1 - out_i0;
  // i-chunk count per launch from a wave model: CTAs are equal-length
  // (one tile column over chunk + 2R planes), one resident per SM, so a launch
  // takes ceil(tiles*c / SMs) * (ceil(nout/c) + 2R) plane-times.  Minimising it
  // reproduced the measured best chunking at 768^3 and 1024^3.
  const int sms = num_sms();
  // L2 prefetch (cp.async.bulk.prefetch.tensor) of a plane's boxes and tiles
  // `pf` planes beyond the shared-memory ring (SGB_V7_PREFETCH=pf; default off).
  // Measured (scripts/pf_sweep.py, alternating order): the fresh (MODE 4)
  // gather gains 1.6-3.7 % at n = 512..1088 (768^3: 1.918 -> 1.846 ms) but
  // loses 9 % at n = 1024 (rows a multiple of 4 KiB: ncu DRAM reads +46 %,
  // the prefetched lines are evicted before their TMA load); the
  // accumulating gather (two tiles per plane) loses 19 % at 768^3 (boxes
  // only: 4 %).  No BASELINE configuration gains, so the default stays off.
  const int pf = (int)std::max<long long>(0, std::min<long long>(8, opt(OPT_V7_PREFETCH, 0)));
  auto chunking = [&](Opt knob, long long tiles) {
    int c = (int)std::max<long long>(0, opt(knob, 0));
    if (c == 0) {
      long long best = -1;
      for (int cc = 1; cc <= 64 && cc <= nout; cc++) {
        const long long len = (nout + cc - 1) / cc;
        const long long waves = (tiles * cc + sms - 1) / sms;
        const long long cost = waves * (len + 2 * Tl::R);
        if (best < 0 || cost < best) best = cost, c = cc;
      }
    }
    const int len = (int)((nout + c - 1) / c);
    return std::make_pair(len, (unsigned)((nout + len - 1) / len));
  };
  const auto ci = chunking(OPT_ICHUNKS, tm.n_interior());
  const auto cf = chunking(OPT_ICHUNKS_F, tm.n_frame());
  // one launch for partial plane ranges (z-slabs, edge bands: measured 5-12%
  // faster there, fewer CTA waves); two launches for the full grid (faster in
  // the sustained single-GPU run); SGB_V7_UNIFIED / SGB_V7_SPLIT force either
  if (peer) {  // fused halo: one launch, halo planes from the neighbours' arrays
    if (!ubwin) {
      set_error(std::string(name) + ": peer halo path needs 16-byte aligned arrays");
      return SGB_EINVAL;
    }
    const auto cu = chunking(OPT_ICHUNKS, (long long)tm.tiles_k * tm.tiles_j);
    star3_v7_unified_peer<MODE, true>
        <<<dim3((unsigned)(tm.tiles_k * tm.tiles_j), cu.second), Tl::THREADS, Tl::SMEM, s>>>(
            maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], c_b, u_1_b, u_2_b, (int)g.n,
            (int)g.i_base, (int)lo, (int)hi, (int)out_i0, (int)out_i1, cu.first, tm, D, pf, *peer);
    return launch_status(name);
  }
  const bool partial = out_i0 != 0 || out_i1 != g.n;
  // v8 interior (below) for the fresh form at n >= 512
  const bool v8 = (MODE == 2 || MODE == 4) && opt(OPT_V8_INTERIOR, MODE == 4 && g.n >= 512) != 0;
  // partial plane ranges (z-slabs, edge bands) take one unified v7 launch
  // (fewer CTA waves) -- except when the interior runs v8: the split launch
  // then wins for slabs too (cfg 5 per-rank step at N = 2 / 4 / 8: 0.99 /
  // 0.94 / 0.87 of single-GPU/N against 0.96 / 0.89 / 0.84 unified,
  // scripts/cfg5_rank_time.py); both give the same bits
  const bool unified =
      opt_flag(OPT_V7_UNIFIED) || (partial && !opt_flag(OPT_V7_SPLIT) && !(v8 && ubwin));
  if (ubwin && unified) {
    const auto cu = chunking(OPT_ICHUNKS, (long long)tm.tiles_k * tm.tiles_j);
    star3_v7_unified<MODE, true>
        <<<dim3((unsigned)(tm.tiles_k * tm.tiles_j), cu.second), Tl::THREADS, Tl::SMEM, s>>>(
            maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], c_b, u_1_b, u_2_b, (int)g.n,
            (int)g.i_base, (int)lo, (int)hi, (int)out_i0, (int)out_i1, cu.first, tm, D, pf);
    return launch_status(name);
  }
  if constexpr (MODE == 2 || MODE == 4) {
    // v8 (bitwise = v7): 24 % fewer instructions, 18 % fewer shared
    // wavefronts, and for the fresh form the c / u_b boxes requested a plane
    // earlier (split stage barriers): the 1024^3 fresh gather 4.61 -> 4.44 ms
    // at burst clocks, 5.26 -> 5.17 ms under the power cap, 768^3 1.93 ->
    // 1.87 ms; the accumulating form gains < 1 %, small grids lose (n = 200:
    // +5 %), so the default is the fresh form (cfg 5) at n >= 512;
    // SGB_V8_INTERIOR=0|1 forces either (scripts/v8_check.py, cfg5_ab.py).
    // SGB_V8_FRAME=1: the frame tiles in v8 too (bitwise the same; 1024^3
    // 4.62 -> 4.54 ms but 768^3 1.87 -> 1.92 ms, so off by default).
    if (tm.n_interior() > 0 && ubwin && v8) {
      using T8 = StarTile8<MODE>;
      if (int r = ensure_smem((const void*)star3_v8_kernel<MODE>, T8::SMEM, name)) return r;
      auto launch8 = [&](int which, unsigned ctas, std::pair<int, unsigned> c) {
        star3_v8_kernel<MODE><<<dim3(ctas, c.second), T8::THREADS, T8::SMEM, s>>>(
            maps[0], maps[1], maps[2], maps[3], maps[4], c_b, u_1_b, (int)g.n, (int)g.i_base,
            (int)lo, (int)hi, (int)out_i0, (int)out_i1, c.first, tm, D, which);
        return launch_status(name);
      };
      if (tm.n_frame() > 0) {
        if (opt_flag(OPT_V8_FRAME)) {
          if (int st = launch8(1, (unsigned)tm.n_frame(), cf)) return st;
        } else {
          star3_v7_kernel<MODE, false, true>
              <<<dim3((unsigned)tm.n_frame(), cf.second), Tl::THREADS, Tl::SMEM, s>>>(
                  maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], c_b, u_1_b, u_2_b,
                  (int)g.n, (int)g.i_base, (int)lo, (int)hi, (int)out_i0, (int)out_i1,
                  cf.first, tm, D, pf);
          if (int st = launch_status(name)) return st;
        }
      }
      // balanced last wave (star3_v8_balanced): one chunk per column, more
      // tiles than SMs and a partly filled last wave that the model prices
      // >= 2 % above the balanced schedule
      const long long T = tm.n_interior();
      const long long rem = T % sms, nfill = sms - rem;
      if (ci.second == 1 && T > sms && rem > 0 && opt(OPT_V8_BALANCE, 1) != 0) {
        const long long ppf = (rem + nfill - 1) / nfill;  // pieces per filler CTA
        // rem CTAs run m + 2R planes, fillers ppf * (nout - m + 2R): equal at
        long long m = (ppf * (nout + 2 * Tl::R) - 2 * Tl::R) / (ppf + 1);
        if (opt(OPT_V8_BALANCE, 1) > 1) m = opt(OPT_V8_BALANCE, 1);  // forced split (sweeps)
        m = std::max<long long>(1, std::min<long long>(m, nout - 1));
        const long long bal = (T / sms) * (nout + 2 * Tl::R) +
                              std::max(m + 2 * Tl::R, ppf * (nout - m + 2 * Tl::R));
        const long long plain = ((T + sms - 1) / sms) * (nout + 2 * Tl::R);
        if (bal * 100 <= plain * 98) {
          if (int r = ensure_smem((const void*)star3_v8_balanced<MODE>, T8::SMEM, name)) return r;
          star3_v8_balanced<MODE><<<dim3((unsigned)(T + nfill)), T8::THREADS, T8::SMEM, s>>>(
              maps[0], maps[1], maps[2], maps[3], maps[4], c_b, u_1_b, (int)g.n, (int)g.i_base,
              (int)lo, (int)hi, (int)out_i0, (int)out_i1, tm, D, (int)(T - rem), (int)rem,
              (int)(out_i0 + m));
          return launch_status(name);
        }
      }
      return launch8(0, (unsigned)tm.n_interior(), ci);
    }
  }
  // Frame launch on a side stream, concurrent with the interior launch
  // (SGB_FORK=1): an A/B with alternating order (scripts/cfg5_ab.py) measured
  // it slower at 1024^3 (4.75 vs 4.67 ms) and 768^3 (1.99 vs 1.86 ms), so the
  // default is one stream.
  const long long fork_opt = opt(OPT_FORK, 0);
  const bool fork = tm.n_interior() > 0 && tm.n_frame() > 0 && fork_opt > 0;
  SideStream* ss = fork ? side_stream() : nullptr;
  if (ss) {
    if (cudaEventRecord(ss->fork, s) != cudaSuccess ||
        cudaStreamWaitEvent(ss->s, ss->fork, 0) != cudaSuccess)
      return launch_status(name);
  }
  if (tm.n_frame() > 0) {
    auto k = ubwin ? star3_v7_kernel<MODE, false, true> : star3_v7_kernel<MODE, false, false>;
    k<<<dim3((unsigned)tm.n_frame(), cf.second), Tl::THREADS, Tl::SMEM, ss ? ss->s : s>>>(
        maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], c_b, u_1_b, u_2_b, (int)g.n,
        (int)g.i_base, (int)lo, (int)hi, (int)out_i0, (int)out_i1, cf.first, tm, D, pf);
    const int st = launch_status(name);
    if (st) return st;
  }
  if (tm.n_interior() > 0) {
    auto k = ubwin ? star3_v7_kernel<MODE, true, true> : star3_v7_kernel<MODE, true, false>;
    k<<<dim3((unsigned)tm.n_interior(), ci.second), Tl::THREADS, Tl::SMEM, s>>>(
        maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], c_b, u_1_b, u_2_b, (int)g.n,
        (int)g.i_base, (int)lo, (int)hi, (int)out_i0, (int)out_i1, ci.first, tm, D, pf);
    const int st = launch_status(name);
    if (st) return st;
  }
  if (ss) {
    if (cudaEventRecord(ss->join, ss->s) != cudaSuccess ||
        cudaStreamWaitEvent(s, ss->join, 0) != cudaSuccess)
      return launch_status(name);
  }
  return 0;
}


// Local arrays hold exactly the global planes [g.i_base, g.i_base + g.nplanes);
// neighbour side k (0 lower, 1 upper) holds planes [nb_base[k], nb_base[k] +
// nb_np[k]) of arrays nb_c / nb_u1 / nb_ub (nullptr: no neighbour, grid end).
template <int MODE>
inline int star3_v7_gather_peer(const Slab3& g, long long lo, long long hi, long long out_i0,
                                long long out_i1, float D, const float* c, float* c_b,
                                const float* u_1, float* u_1_b, const float* u_b,
                                const float* const nb_c[2], const float* const nb_u1[2],
                                const float* const nb_ub[2], const int nb_base[2],
                                const int nb_np[2], cudaStream_t s, const char* name) {
  using Tl = StarTile7<MODE>;
  constexpr int R = Tl::R;
  PeerHalo ph;
  std::memset(&ph, 0, sizeof(ph));
  ph.own0 = (int)g.i_base;
  ph.own1 = (int)(g.i_base + g.nplanes);
  for (int k = 0; k < 2; k++) {
    if (!nb_c[k]) continue;
    if (!nb_u1[k] || !nb_ub[k] || nb_np[k] <= 0) return SGB_EINVAL;
    ph.has[k] = 1;
    ph.base[k] = nb_base[k];
    int rc = encode_3d(&ph.c[k], nb_c[k], g.n, nb_np[k], Tl::BW, Tl::BJ, name);
    rc |= encode_3d(&ph.u1[k], nb_u1[k], g.n, nb_np[k], Tl::BW, Tl::BJ, name);
    const int w = encode_3d_window(&ph.ub[k], nb_ub[k], g.n, nb_np[k], lo, hi - lo + 1, Tl::BW,
                                   Tl::BJ, name);
    if (rc || w != 0) {
      set_error(std::string(name) + ": peer maps (16-byte aligned neighbour arrays needed)");
      return SGB_EINVAL;
    }
  }
  // every input plane the outputs need must be held locally or by a neighbour
  const long long need_lo = std::max<long long>(0, out_i0 - R);
  const long long need_hi = std::min<long long>(g.n - 1, out_i1 - 1 + R);
  for (long long p = need_lo; p <= need_hi; p++) {
    const bool local = p >= ph.own0 && p < ph.own1;
    const bool low = ph.has[0] && p < ph.own0 && p >= ph.base[0] && p < ph.base[0] + nb_np[0];
    const bool up = ph.has[1] && p >= ph.own1 && p >= ph.base[1] && p < ph.base[1] + nb_np[1];
    if (!local && !low && !up) {
      set_error(std::string(name) + ": input plane " + std::to_string(p) +
                " held by no rank (local + neighbours must cover the R halo)");
      return SGB_EINVAL;
    }
  }
  if (out_i0 < ph.own0 || out_i1 > ph.own1) return SGB_EINVAL;
  return star3_v7_gather<MODE>(g, lo, hi, out_i0, out_i1, D, c, c_b, u_1, u_1_b, nullptr, u_b, s,
                               name, &ph);
}

}  // namespace sgb
