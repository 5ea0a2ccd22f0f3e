// Streaming primal for the 3D star families (sm_100a; fp32, TMA path).
//
// run_nest semantics (interp.cpp:153-173; emitted form codegen.cpp:311-330):
// on the primal box B = [lo, hi]^3
//     u = 2 u_1 - u_2 + c^(1|2) D Lap_R(u_1)        (WAVE3D_C / _C2 / R4)
// points outside B untouched.  Same streaming scheme as the radius-4 gather
// kernel (star3d_r4.cuh): a 64 (k) x 32 (j) column tile per CTA streams over i
// through a 3-stage TMA ring; per plane p the ring holds the u_1 halo box of
// p and the c, u_2, u_1 tiles of the output plane o = p - R; each thread owns
// 2 rows x 4 k points and keeps the i direction in 2R+1 rotating float4
// accumulators (field2x4), so Lap(u_1)[o] is complete when plane p = o + R
// has been read.  256 threads, ~108 KB smem: 2 CTAs per SM.  Algorithmic
// traffic 16 B/pt (c, u_1, u_2 read; u written).
#pragma once

#include "star3d_r4.cuh"

namespace sgb {

template <int MODE>
struct PrimalTile {
  static constexpr int R = Star3<MODE>::R;
  static constexpr int TK = 64, TJ = 32, HK = 4, HJ = R;
  static constexpr int BW = TK + 2 * HK;  // 72 (field2x4's row pitch)
  static constexpr int BJ = TJ + 2 * HJ;
  static constexpr int RING = 2 * R + 1;
  static constexpr int NS = 3;
  static constexpr int THREADS = 16 * (TJ / 2);  // 2 rows x 4 k per thread
  static constexpr int BOX_BYTES = BW * BJ * 4;
  static constexpr int BF = ((BOX_BYTES + 127) / 128) * 128 / 4;
  static constexpr int TILE = TK * TJ;
  static constexpr int NT = Star3<MODE>::kIncrement ? 4 : 3;  // c, u_2, u_1 (, u)
  static constexpr int SF = BF + NT * TILE;
  static constexpr int SMEM = NS * SF * 4 + NS * 8;
  static_assert(RING % NS == 0, "static stage index");
  static_assert(BW == 72, "field2x4 row pitch");
};

template <int MODE>
__global__ void __launch_bounds__(PrimalTile<MODE>::THREADS, 2)
    star3_primal_tma_kernel(const __grid_constant__ CUtensorMap tm_box,
                            const __grid_constant__ CUtensorMap tm_c,
                            const __grid_constant__ CUtensorMap tm_u2,
                            const __grid_constant__ CUtensorMap tm_u1,
                            const __grid_constant__ CUtensorMap tm_u, float* __restrict__ u,
                            int n, int lo, int hi, int chunk, int tiles_k, float D) {
  using Tl = PrimalTile<MODE>;
  using S3 = Star3<MODE>;
  constexpr int R = Tl::R, HJ = Tl::HJ, HK = Tl::HK, TK = Tl::TK, RING = Tl::RING;
  constexpr int NS = Tl::NS, BF = Tl::BF, TILE = Tl::TILE, SF = Tl::SF, NT = Tl::NT;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);  // [NS][box | c | u_2 | u_1 (| u)]
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
    float* dst = stage + s * SF;
    const int p = pstart + it;
    const bool emit = it >= 2 * R;
    tma::mbar_arrive_expect_tx(&bars[s], Tl::BOX_BYTES + (emit ? NT * TILE * 4 : 0));
    tma::load_3d(dst, &tm_box, &bars[s], k0 - HK, j0 - HJ, p);
    if (emit) {
      const int o = p - R;
      tma::load_3d(dst + BF, &tm_c, &bars[s], k0, j0, o);
      tma::load_3d(dst + BF + TILE, &tm_u2, &bars[s], k0, j0, o);
      tma::load_3d(dst + BF + 2 * TILE, &tm_u1, &bars[s], k0, j0, o);
      if (NT == 4) tma::load_3d(dst + BF + 3 * TILE, &tm_u, &bars[s], k0, j0, o);
    }
  };
  if (tid == 0)
    for (int it = 0; it < NS && it < P; it++) issue(it);

  const int jr0 = j0 + 2 * ty, kc = k0 + 4 * tx;
  const int r0 = 2 * ty + HJ, col = HK + 4 * tx;
  const int trow = 2 * ty * TK + 4 * tx;
  const long long plane = (long long)n * n;
  const int coff = jr0 * n + kc;
  const bool tile_in = j0 >= lo && j0 + Tl::TJ - 1 <= hi && k0 >= lo && k0 + TK - 1 <= hi;
  bool jin[2], kin[4];
#pragma unroll
  for (int h = 0; h < 2; h++) jin[h] = jr0 + h >= lo && jr0 + h <= hi;
#pragma unroll
  for (int m = 0; m < 4; m++) kin[m] = kc + m >= lo && kc + m <= hi;
  const bool kall = kin[0] && kin[3] && kc + 3 < n;  // all 4 k points written: one 16-byte store

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
        const float* F = stage + s * SF;
        tma::mbar_wait(&bars[s], (par0 + ph / NS) & 1);
        field2x4<R, RING>(F, r0, col, w0, wr, acc, ph);
        if (it >= 2 * R) {
          const int es = (ph + R + 1) % RING;
          const int o = pstart + it - R;
          float* urow = u + (long long)o * plane + coff;
#pragma unroll
          for (int h = 0; h < 2; h++) {
            const float4 cv = lds4(F + BF + trow + h * TK);
            const float4 u2 = lds4(F + BF + TILE + trow + h * TK);
            const float4 u1 = lds4(F + BF + 2 * TILE + trow + h * TK);
            const float4 cc = S3::kC2 ? mul4(cv, cv) : cv;
            // (2 u_1 - u_2) + (cc D) Lap, the generic kernel's grouping
            float4 v = add4(fmas4(2.f, u1, muls4(-1.f, u2)), mul4(muls4(D, cc), acc[es][h]));
            if (NT == 4) v = add4(lds4(F + BF + 3 * TILE + trow + h * TK), v);
            if (tile_in || (jin[h] && kall)) {
              __stcs(reinterpret_cast<float4*>(urow + h * n), v);
            } else if (jin[h]) {
              const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
              for (int m = 0; m < 4; m++)
                if (kin[m] && kc + m < n) urow[h * n + m] = vv[m];
            }
          }
        }
        __syncthreads();  // stage s consumed by every thread
        if (tid == 0 && it + NS < P) issue(it + NS);
      }
    }
  }
}

// Host launcher; returns 1 when the TMA path does not apply (caller falls
// back to the per-point kernel), 0 / negative like the other entries.
template <int MODE>
inline int star3_primal_tma(long long n, float D, const float* c, const float* u_1,
                            const float* u_2, float* u, cudaStream_t s, const char* name) {
  using Tl = PrimalTile<MODE>;
  constexpr int R = Tl::R;
  const long long lo = R, hi = n - 1 - R;
  if (n % 4 != 0 || n < 2 * R + 1 || n > (1 << 20)) return 1;
  for (const void* p : {(const void*)c, (const void*)u_1, (const void*)u_2, (const void*)u})
    if (reinterpret_cast<uintptr_t>(p) & 15) return 1;
  CUtensorMap maps[5];
  int rc = 0;
  rc |= encode_3d(&maps[0], u_1, n, n, Tl::BW, Tl::BJ, name);
  rc |= encode_3d(&maps[1], c, n, n, Tl::TK, Tl::TJ, name);
  rc |= encode_3d(&maps[2], u_2, n, n, Tl::TK, Tl::TJ, name);
  rc |= encode_3d(&maps[3], u_1, n, n, Tl::TK, Tl::TJ, name);
  rc |= encode_3d(&maps[4], u, n, n, Tl::TK, Tl::TJ, name);
  if (rc) return SGB_EINVAL;
  if (int rc = ensure_smem((const void*)star3_primal_tma_kernel<MODE>, Tl::SMEM, name))
    return rc;
  const int tiles_k = (int)((n + Tl::TK - 1) / Tl::TK);
  const long long tiles = (long long)tiles_k * ((n + Tl::TJ - 1) / Tl::TJ);
  const long long nout = hi - lo + 1;
  // wave model (star3d_r4.cuh): 2 CTAs per SM, equal-length CTAs
  const long long slots = 2LL * num_sms();
  int nch = 1;
  long long best = -1;
  for (int cc = 1; cc <= 64 && cc <= nout; cc++) {
    const long long len = (nout + cc - 1) / cc;
    const long long cost = ((tiles * cc + slots - 1) / slots) * (len + 2 * R);
    if (best < 0 || cost < best) best = cost, nch = cc;
  }
  // Radius 4: short chunks (~48 planes) keep the resident CTAs streaming
  // nearly the same planes, so the u_1 halo rows a tile shares with its
  // neighbours and the u_1 centre tile (re-read R planes after its box) are
  // still in L2: 768^3 1.34 -> 1.11 ms although every chunk re-reads 2R halo
  // planes.  Radius 1 keeps the wave model (measured best there).
  if (R >= 2) nch = (int)std::max<long long>(nch, (nout + 47) / 48);
  if (opt(OPT_PRIMAL_CHUNKS, 0) > 0) nch = (int)opt(OPT_PRIMAL_CHUNKS, 0);
  const int chunk = (int)((nout + nch - 1) / nch);
  const unsigned gy = (unsigned)((nout + chunk - 1) / chunk);
  star3_primal_tma_kernel<MODE><<<dim3((unsigned)tiles, gy), Tl::THREADS, Tl::SMEM, s>>>(
      maps[0], maps[1], maps[2], maps[3], maps[4], u, (int)n, (int)lo, (int)hi, chunk, tiles_k,
      D);
  return launch_status(name);
}

}  // namespace sgb
