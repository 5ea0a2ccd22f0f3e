// Device-side synthetic input generation (BASELINE.json distributions).
//
// Counter-based: every value is a pure function of (seed, stream_id, global
// flat index), so slabs of any z-decomposition regenerate exactly the values
// a single GPU would hold -- the property the multi-GPU runs rely on to be
// compared against one oracle output.
#include "sgb_common.cuh"

namespace sgb {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

__host__ __device__ __forceinline__ uint64_t hash_key(uint64_t seed, uint64_t stream) {
  return seed * 0x9E3779B97F4A7C15ull + mix64(stream + 0xD1B54A32D192ED03ull);
}
__device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return mix64(hash_key(seed, stream) + ctr);
}

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {  // murmur3 finaliser
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}

// One Box-Muller pair from the hash of pair index m: (cos branch, sin branch)
// = the values of flat indices 2m and 2m+1.  Built for the XU (MUFU) pipe
// and issue rate, since the generator runs inside cfg 5's timed step (the
// 64-bit splitmix + IEEE form was issue-bound, then the two-murmur3 form
// MUFU/I2F-throttled at ~33 instructions per value, profiles/):
//   * one murmur3 finaliser per pair, keyed by the 64-bit stream key; the
//     angle's bits are its Fibonacci-lattice partner a * 0x9E3779B9 (an odd
//     multiplier: a permutation of a, whose top 23 bits are equidistributed
//     against a's -- the 2D golden-ratio lattice, sampled at hashed points);
//   * uniforms from the mantissa bits (OR into an exponent, one FADD)
//     instead of I2F conversions, which share the XU pipe with MUFU;
//   * MUFU lg2 / sqrt / sin / cos (flush-to-zero approximations; the angle in
//     [-pi, pi), where sin.approx / cos.approx are accurate): 2 XU ops per value.
struct NormalPair {
  float rad, cs, sn;  // value(2m) = rad * cs, value(2m+1) = rad * sn
};
__device__ __forceinline__ NormalPair normal_pair_polar(uint64_t key, uint64_t m) {
  const uint32_t a = fmix32((uint32_t)m ^ (uint32_t)key ^ ((uint32_t)(m >> 32) * 0x9E3779B9u));
  const uint32_t b = (a ^ (uint32_t)(key >> 32)) * 0x9E3779B9u;
  const float u1 = 2.0f - __uint_as_float((a >> 9) | 0x3F800000u);            // (0, 1]
  const float th = fmaf(__uint_as_float((b >> 9) | 0x40000000u), 3.14159265358979f,
                        -9.42477796076938f);                                   // [-pi, pi)
  float l2, rad, sn, cs;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"(u1));
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(rad) : "f"(-1.3862943611198906f * l2));  // -2 ln u1
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(sn) : "f"(th));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(cs) : "f"(th));
  return NormalPair{rad, cs, sn};
}
__device__ __forceinline__ float2 normal_pair(uint64_t key, uint64_t m) {
  const NormalPair p = normal_pair_polar(key, m);
  return make_float2(p.rad * p.cs, p.rad * p.sn);
}

// kind 0: N(mean, scale^2); kind 1: U[mean, mean + scale).
// Normals come in Box-Muller pairs: indices 2m and 2m+1 share the hash of m
// (cos / sin branch), so value(index) is still a pure function of the index.
__device__ __forceinline__ double draw(uint64_t seed, uint64_t stream, uint64_t idx, int kind) {
  if (kind == 1) return (double)(hash3(seed, stream, idx) >> 11) * 0x1.0p-53;
  const float2 z = normal_pair(hash_key(seed, stream), idx >> 1);
  return (double)((idx & 1) ? z.y : z.x);
}

template <typename T>
__global__ void fill_random_kernel(T* dst, long long count, long long base, uint64_t seed,
                                   uint64_t stream, int kind, double mean, double scale) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x) {
    const double z = draw(seed, stream, (uint64_t)(base + t), kind);
    dst[t] = (T)(mean + scale * z);
  }
}

// 3D fill with a fused zero halo: planes [i_base, i_base+nplanes) of an n^3
// grid, h-point zero shell, N(mean, scale^2) elsewhere; 4 points per thread.
// With n even the 4 points are two whole Box-Muller pairs, each computed once
// (same values as draw()).  32-bit coordinates (n <= 2^20), a 64-bit flat
// index advanced per plane.
// T = float, or double holding the SAME (fp32) values widened: the fp64
// configurations regenerate exactly the inputs of the fp32 ones.
template <typename T>
__global__ void fill_normal3d_kernel(T* dst, int n, int i_base, int nplanes, int h,
                                     uint64_t seed, uint64_t stream, float mean, float scale) {
  const int k = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int j = blockIdx.y;
  if (k >= n) return;
  const uint64_t key = hash_key(seed, stream);
  const bool jh = j < h || j >= n - h;
  const bool kin = k >= h && k + 3 < n - h;  // no k halo point among the 4
  const long long plane = (long long)n * n;
  const long long dg = (long long)gridDim.z * plane;
  long long g = ((long long)(i_base + (int)blockIdx.z) * n + j) * n + k;  // global flat index
  T* p = dst + ((long long)blockIdx.z * n + j) * n + k;
  const long long dp = dg;
  for (int li = blockIdx.z; li < nplanes; li += gridDim.z, g += dg, p += dp) {
    const int i = i_base + li;
    const bool rowh = jh || i < h || i >= n - h;
    float v[4];
    if ((g & 1) == 0 && k + 3 < n) {  // two whole pairs
      const NormalPair a = normal_pair_polar(key, (uint64_t)g >> 1);
      const NormalPair b = normal_pair_polar(key, ((uint64_t)g >> 1) + 1);
      // fmaf(scale * rad, cos|sin, mean): the pair kernel's formula (bitwise
      // equal values; = rad * cos|sin, the draw() value, at mean 0, scale 1)
      const float z[4] = {fmaf(scale * a.rad, a.cs, mean), fmaf(scale * a.rad, a.sn, mean),
                          fmaf(scale * b.rad, b.cs, mean), fmaf(scale * b.rad, b.sn, mean)};
#pragma unroll
      for (int m = 0; m < 4; m++) {
        const int kk = k + m;
        v[m] = (rowh || kk < h || kk >= n - h) ? 0.f : z[m];
      }
    } else {
#pragma unroll
      for (int m = 0; m < 4; m++) {
        const int kk = k + m;
        const bool halo = rowh || kk < h || kk >= n - h;
        v[m] = (halo || kk >= n) ? 0.f
                                 : mean + scale * (float)draw(seed, stream, (uint64_t)(g + m), 0);
      }
    }
    if (n % 4 == 0) {
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
        *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
      }
    } else {
      for (int m = 0; m < 4 && k + m < n; m++) p[m] = v[m];
    }
  }
}

// Two fields of one step in ONE pass (cfg 5 regenerates u_1 and the seed u_b
// every step): fields f = 0, 1 with their own stream key and zero shell h_f,
// N(mean, scale^2) elsewhere -- bitwise the values of two fill_normal3d calls
// (value(2m) = mean + scale * rad * cs is evaluated as fmaf(scale * rad, cs,
// mean) there too).  Fast-path shapes only: n % 4 == 0 (so a thread's 4
// consecutive k are two whole Box-Muller pairs) and 16-byte aligned arrays;
// the entry falls back to two fill_normal3d_kernel launches otherwise.  Each
// thread owns 4 consecutive k of one row of both fields and strides over
// planes: 8 values, 4 pairs in flight, two 16-byte (fp32) stores per plane.
template <typename T>
__global__ void __launch_bounds__(128) fill_normal3d_pair_kernel(
    T* __restrict__ d0, T* __restrict__ d1, int n, int i_base, int nplanes, int h0, int h1,
    uint64_t key0, uint64_t key1, float mean, float scale) {
  const int k = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int j = blockIdx.y;
  if (k >= n) return;
  // plane-independent parts of the zero-shell masks: bit m = point k+m inside
  uint32_t km0 = 0, km1 = 0;
#pragma unroll
  for (int m = 0; m < 4; m++) {
    if (k + m >= h0 && k + m < n - h0) km0 |= 1u << m;
    if (k + m >= h1 && k + m < n - h1) km1 |= 1u << m;
  }
  const bool j0h = j < h0 || j >= n - h0, j1h = j < h1 || j >= n - h1;
  const long long plane = (long long)n * n;
  const long long dg = (long long)gridDim.z * plane;
  long long g = ((long long)(i_base + (int)blockIdx.z) * n + j) * n + k;  // global flat index
  long long off = ((long long)blockIdx.z * n + j) * n + k;
  for (int li = blockIdx.z; li < nplanes; li += gridDim.z, g += dg, off += dg) {
    const int i = i_base + li;
    const uint64_t m = (uint64_t)g >> 1;
    const NormalPair a0 = normal_pair_polar(key0, m), b0 = normal_pair_polar(key0, m + 1);
    const NormalPair a1 = normal_pair_polar(key1, m), b1 = normal_pair_polar(key1, m + 1);
    const float z0[4] = {fmaf(scale * a0.rad, a0.cs, mean), fmaf(scale * a0.rad, a0.sn, mean),
                         fmaf(scale * b0.rad, b0.cs, mean), fmaf(scale * b0.rad, b0.sn, mean)};
    const float z1[4] = {fmaf(scale * a1.rad, a1.cs, mean), fmaf(scale * a1.rad, a1.sn, mean),
                         fmaf(scale * b1.rad, b1.cs, mean), fmaf(scale * b1.rad, b1.sn, mean)};
    const uint32_t m0 = (j0h || i < h0 || i >= n - h0) ? 0u : km0;
    const uint32_t m1 = (j1h || i < h1 || i >= n - h1) ? 0u : km1;
    float v0[4], v1[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      v0[q] = (m0 >> q) & 1 ? z0[q] : 0.f;
      v1[q] = (m1 >> q) & 1 ? z1[q] : 0.f;
    }
    if constexpr (sizeof(T) == 4) {
      __stcs(reinterpret_cast<float4*>(d0 + off), make_float4(v0[0], v0[1], v0[2], v0[3]));
      __stcs(reinterpret_cast<float4*>(d1 + off), make_float4(v1[0], v1[1], v1[2], v1[3]));
    } else {
      __stcs(reinterpret_cast<double2*>(d0 + off), make_double2(v0[0], v0[1]));
      __stcs(reinterpret_cast<double2*>(d0 + off + 2), make_double2(v0[2], v0[3]));
      __stcs(reinterpret_cast<double2*>(d1 + off), make_double2(v1[0], v1[1]));
      __stcs(reinterpret_cast<double2*>(d1 + off + 2), make_double2(v1[2], v1[3]));
    }
  }
}

// fp64 form of the pair kernel: each thread owns ONE Box-Muller pair (2
// consecutive k) of both fields, so a warp's 16-byte stores cover 512
// contiguous bytes per field.  (Four k per thread, as in the fp32 kernel,
// left every double2 store instruction writing half of each 32-byte sector,
// the other half by the next instruction: 3.7 TB/s at 1024^3.)  Same values.
__global__ void __launch_bounds__(128) fill_normal3d_pair_f64_kernel(
    double* __restrict__ d0, double* __restrict__ d1, int n, int i_base, int nplanes, int h0,
    int h1, uint64_t key0, uint64_t key1, float mean, float scale) {
  const int k = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int j = blockIdx.y;
  if (k >= n) return;
  uint32_t km0 = 0, km1 = 0;
#pragma unroll
  for (int m = 0; m < 2; m++) {
    if (k + m >= h0 && k + m < n - h0) km0 |= 1u << m;
    if (k + m >= h1 && k + m < n - h1) km1 |= 1u << m;
  }
  const bool j0h = j < h0 || j >= n - h0, j1h = j < h1 || j >= n - h1;
  const long long plane = (long long)n * n;
  const long long dg = (long long)gridDim.z * plane;
  long long g = ((long long)(i_base + (int)blockIdx.z) * n + j) * n + k;  // global flat index
  long long off = ((long long)blockIdx.z * n + j) * n + k;
  for (int li = blockIdx.z; li < nplanes; li += gridDim.z, g += dg, off += dg) {
    const int i = i_base + li;
    const uint64_t m = (uint64_t)g >> 1;
    const NormalPair a0 = normal_pair_polar(key0, m), a1 = normal_pair_polar(key1, m);
    const float z0[2] = {fmaf(scale * a0.rad, a0.cs, mean), fmaf(scale * a0.rad, a0.sn, mean)};
    const float z1[2] = {fmaf(scale * a1.rad, a1.cs, mean), fmaf(scale * a1.rad, a1.sn, mean)};
    const uint32_t m0 = (j0h || i < h0 || i >= n - h0) ? 0u : km0;
    const uint32_t m1 = (j1h || i < h1 || i >= n - h1) ? 0u : km1;
    __stcs(reinterpret_cast<double2*>(d0 + off),
           make_double2(m0 & 1 ? z0[0] : 0.f, m0 & 2 ? z0[1] : 0.f));
    __stcs(reinterpret_cast<double2*>(d1 + off),
           make_double2(m1 & 1 ? z1[0] : 0.f, m1 & 2 ? z1[1] : 0.f));
  }
}

template <typename T>
__global__ void zero_halo_kernel(T* a, int d, long long n, int h, long long i_base,
                                 long long nplanes) {
  const long long per = (d == 3) ? n * n : (d == 2 ? n : 1);
  const long long total = nplanes * per;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long li = t / per, rem = t % per;
    const long long i = i_base + li;
    bool halo = i < h || i >= n - h;
    if (d >= 2) {
      const long long j = (d == 3) ? rem / n : rem;
      halo |= j < h || j >= n - h;
      if (d == 3) {
        const long long k = rem % n;
        halo |= k < h || k >= n - h;
      }
    }
    if (halo) a[t] = T(0);
  }
}

__global__ void layered_kernel(float* c, long long n, int layers, double lo, double hi,
                               uint64_t seed, long long i_base, long long nplanes) {
  const long long total = nplanes * n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long i = i_base + t / (n * n);
    const long long layer = (i * layers) / n;
    c[t] = (float)(lo + (hi - lo) * draw(seed, 0x1A7E5ull, (uint64_t)layer, 1));
  }
}

// y[p] += alpha * x[p] on the box [lo, hi]^3 of planes [i_base, i_base+nplanes).
// Each thread owns 4 consecutive k of one row (one 16-byte vector for fp32
// when the 4 lie inside the box and are aligned, else element by element);
// a block covers 256 k x 4 rows, so the grid is ~n^3/1024 blocks.
template <typename T>
__global__ void __launch_bounds__(256) box_axpy_kernel(T* __restrict__ y,
                                                       const T* __restrict__ x, T alpha,
                                                       long long n, long long lo, long long hi,
                                                       long long i_base, long long nplanes) {
  const long long k0 = 4 * (blockIdx.x * 64LL + threadIdx.x);
  const long long j = blockIdx.y * 4LL + threadIdx.y;
  const long long li = blockIdx.z;
  const long long i = i_base + li;
  if (k0 >= n || j >= n || li >= nplanes) return;
  if (i < lo || i > hi || j < lo || j > hi || k0 + 3 < lo || k0 > hi) return;
  const long long t = (li * n + j) * n + k0;
  if (sizeof(T) == 4 && k0 >= lo && k0 + 3 <= hi &&
      ((reinterpret_cast<uintptr_t>(y + t) | reinterpret_cast<uintptr_t>(x + t)) & 15) == 0) {
    float4* yv = reinterpret_cast<float4*>(y + t);
    const float4 xv = __ldcs(reinterpret_cast<const float4*>(x + t));
    float4 v = *yv;
    const float a = (float)alpha;
    v.x += a * xv.x;
    v.y += a * xv.y;
    v.z += a * xv.z;
    v.w += a * xv.w;
    *yv = v;
    return;
  }
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const long long k = k0 + m;
    if (k >= lo && k <= hi && k < n) y[t + m] += alpha * x[t + m];
  }
}

// y = 0 + alpha * x on the box [lo, hi]^3, y = 0 elsewhere, on local planes
// [i_base, i_base+nplanes): a zeroed y followed by box_axpy, in one pass
// (bitwise the same result, the explicit 0 + keeps the sign of zero).
template <typename T>
__global__ void __launch_bounds__(256) box_set_kernel(T* __restrict__ y, const T* __restrict__ x,
                                                      T alpha, long long n, long long lo,
                                                      long long hi, long long i_base,
                                                      long long nplanes) {
  const long long k0 = 4 * (blockIdx.x * 64LL + threadIdx.x);
  const long long j = blockIdx.y * 4LL + threadIdx.y;
  const long long li = blockIdx.z;
  if (k0 >= n || j >= n || li >= nplanes) return;
  const long long i = i_base + li;
  const bool row = i >= lo && i <= hi && j >= lo && j <= hi;
  const long long t = (li * n + j) * n + k0;
#pragma unroll
  for (int m = 0; m < 4; m++) {
    const long long k = k0 + m;
    if (k < n) y[t + m] = (row && k >= lo && k <= hi) ? T(0) + alpha * x[t + m] : T(0);
  }
}

__global__ void smooth5_kernel(const double* src, double* dst, long long n) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long i = blockIdx.y * (long long)blockDim.y + threadIdx.y;
  if (i >= n || j >= n) return;
  const long long x = i * n + j;
  if (i == 0 || j == 0 || i == n - 1 || j == n - 1) {
    dst[x] = src[x];
    return;
  }
  dst[x] = (src[x] + src[x - n] + src[x + n] + src[x - 1] + src[x + 1]) / 5.0;
}

static unsigned fill_grid(long long count) {
  long long g = (count + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  return (unsigned)(g < 1 ? 1 : g);
}

template <typename T>
static int fill_normal3d_pair(const char* name, T* a, int halo_a, uint64_t stream_a, T* b,
                              int halo_b, uint64_t stream_b, int n, int i_base, int nplanes,
                              uint64_t seed, double mean, double scale, cudaStream_t s) {
  if (!a || !b || a == b || n <= 0 || nplanes <= 0 || halo_a < 0 || halo_b < 0 ||
      n > (1 << 20))
  {
    set_error(std::string(name) + ": bad arguments");
    return SGB_EINVAL;
  }
  if (n % 4 != 0 || ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15)) {
    // general shapes: two single-field passes (same values)
    dim3 bl(64), g((unsigned)((n / 4 + 63) / 64 + ((n % 4) ? 1 : 0)), (unsigned)n,
                   (unsigned)(nplanes < 64 ? nplanes : 64));
    fill_normal3d_kernel<T><<<g, bl, 0, s>>>(a, n, i_base, nplanes, halo_a, seed, stream_a,
                                             (float)mean, (float)scale);
    if (int rc = launch_status(name)) return rc;
    fill_normal3d_kernel<T><<<g, bl, 0, s>>>(b, n, i_base, nplanes, halo_b, seed, stream_b,
                                             (float)mean, (float)scale);
    return launch_status(name);
  }
  // 128 threads x 4 k (fp64: 2 k) of one row; planes strided so the grid
  // holds a few waves of 148 SMs x 16 resident blocks and each thread runs
  // several planes
  const int per = sizeof(T) == 8 ? 2 : 4;
  const unsigned gx = (unsigned)((n / per + 127) / 128);
  const long long rows = (long long)gx * n;
  long long gz = (148LL * 16 * 4 + rows - 1) / rows;
  if (gz > nplanes) gz = nplanes;
  if (gz < 1) gz = 1;
  if constexpr (sizeof(T) == 8)
    fill_normal3d_pair_f64_kernel<<<dim3(gx, (unsigned)n, (unsigned)gz), 128, 0, s>>>(
        a, b, n, i_base, nplanes, halo_a, halo_b, hash_key(seed, stream_a),
        hash_key(seed, stream_b), (float)mean, (float)scale);
  else
    fill_normal3d_pair_kernel<T><<<dim3(gx, (unsigned)n, (unsigned)gz), 128, 0, s>>>(
        a, b, n, i_base, nplanes, halo_a, halo_b, hash_key(seed, stream_a),
        hash_key(seed, stream_b), (float)mean, (float)scale);
  return launch_status(name);
}

}  // namespace sgb

using namespace sgb;

extern "C" {

int sgb_fill_random_f32(float* dst, long long count, long long index_base, uint64_t seed,
                        uint64_t stream_id, int kind, double mean, double scale,
                        sgb_stream_t stream) {
  if (!dst || count < 0) return SGB_EINVAL;
  if (count == 0) return 0;
  fill_random_kernel<float><<<fill_grid(count), 256, 0, as_stream(stream)>>>(
      dst, count, index_base, seed, stream_id, kind, mean, scale);
  return launch_status("sgb_fill_random_f32");
}

int sgb_fill_random_f64(double* dst, long long count, long long index_base, uint64_t seed,
                        uint64_t stream_id, int kind, double mean, double scale,
                        sgb_stream_t stream) {
  if (!dst || count < 0) return SGB_EINVAL;
  if (count == 0) return 0;
  fill_random_kernel<double><<<fill_grid(count), 256, 0, as_stream(stream)>>>(
      dst, count, index_base, seed, stream_id, kind, mean, scale);
  return launch_status("sgb_fill_random_f64");
}

int sgb_zero_halo_f32(float* a, int d, int n, int h, int i_base, int nplanes,
                      sgb_stream_t stream) {
  if (!a || d < 1 || d > 3 || n <= 0 || nplanes <= 0) return SGB_EINVAL;
  const long long per = d == 3 ? (long long)n * n : (d == 2 ? n : 1);
  zero_halo_kernel<float><<<fill_grid(per * nplanes), 256, 0, as_stream(stream)>>>(
      a, d, n, h, i_base, nplanes);
  return launch_status("sgb_zero_halo_f32");
}

int sgb_zero_halo_f64(double* a, int d, int n, int h, int i_base, int nplanes,
                      sgb_stream_t stream) {
  if (!a || d < 1 || d > 3 || n <= 0 || nplanes <= 0) return SGB_EINVAL;
  const long long per = d == 3 ? (long long)n * n : (d == 2 ? n : 1);
  zero_halo_kernel<double><<<fill_grid(per * nplanes), 256, 0, as_stream(stream)>>>(
      a, d, n, h, i_base, nplanes);
  return launch_status("sgb_zero_halo_f64");
}

int sgb_fill_normal3d_f32(float* dst, int n, int i_base, int nplanes, int halo, uint64_t seed,
                          uint64_t stream_id, double mean, double scale, sgb_stream_t stream) {
  if (!dst || n <= 0 || nplanes <= 0 || halo < 0) return SGB_EINVAL;
  dim3 b(64), g((unsigned)((n / 4 + 63) / 64 + ((n % 4) ? 1 : 0)), (unsigned)n,
                (unsigned)(nplanes < 64 ? nplanes : 64));
  if (n > (1 << 20)) return SGB_EINVAL;
  fill_normal3d_kernel<float><<<g, b, 0, as_stream(stream)>>>(dst, n, i_base, nplanes, halo,
                                                              seed, stream_id, (float)mean,
                                                              (float)scale);
  return launch_status("sgb_fill_normal3d_f32");
}

int sgb_fill_normal3d_f64(double* dst, int n, int i_base, int nplanes, int halo, uint64_t seed,
                          uint64_t stream_id, double mean, double scale, sgb_stream_t stream) {
  if (!dst || n <= 0 || nplanes <= 0 || halo < 0) return SGB_EINVAL;
  if ((reinterpret_cast<uintptr_t>(dst) & 15) && n % 4 == 0) return SGB_EINVAL;
  dim3 b(64), g((unsigned)((n / 4 + 63) / 64 + ((n % 4) ? 1 : 0)), (unsigned)n,
                (unsigned)(nplanes < 64 ? nplanes : 64));
  if (n > (1 << 20)) return SGB_EINVAL;
  fill_normal3d_kernel<double><<<g, b, 0, as_stream(stream)>>>(dst, n, i_base, nplanes, halo,
                                                               seed, stream_id, (float)mean,
                                                               (float)scale);
  return launch_status("sgb_fill_normal3d_f64");
}

int sgb_fill_normal3d_pair_f32(float* a, int halo_a, uint64_t stream_a, float* b, int halo_b,
                               uint64_t stream_b, int n, int i_base, int nplanes, uint64_t seed,
                               double mean, double scale, sgb_stream_t stream) {
  return fill_normal3d_pair("sgb_fill_normal3d_pair_f32", a, halo_a, stream_a, b, halo_b,
                            stream_b, n, i_base, nplanes, seed, mean, scale, as_stream(stream));
}

int sgb_fill_normal3d_pair_f64(double* a, int halo_a, uint64_t stream_a, double* b, int halo_b,
                               uint64_t stream_b, int n, int i_base, int nplanes, uint64_t seed,
                               double mean, double scale, sgb_stream_t stream) {
  return fill_normal3d_pair("sgb_fill_normal3d_pair_f64", a, halo_a, stream_a, b, halo_b,
                            stream_b, n, i_base, nplanes, seed, mean, scale, as_stream(stream));
}

int sgb_fill_layered_f32(float* c, int n, int layers, double lo, double hi, uint64_t seed,
                         int i_base, int nplanes, sgb_stream_t stream) {
  if (!c || n <= 0 || layers <= 0 || nplanes <= 0) return SGB_EINVAL;
  layered_kernel<<<fill_grid((long long)nplanes * n * n), 256, 0, as_stream(stream)>>>(
      c, n, layers, lo, hi, seed, i_base, nplanes);
  return launch_status("sgb_fill_layered_f32");
}

int sgb_box_axpy_f32(float* y, const float* x, double alpha, int n, int lo, int hi, int i_base,
                     int nplanes, sgb_stream_t stream) {
  if (!y || !x || n <= 0 || nplanes <= 0) return SGB_EINVAL;
  dim3 g((unsigned)((n + 255) / 256), (unsigned)((n + 3) / 4), (unsigned)nplanes);
  box_axpy_kernel<float><<<g, dim3(64, 4), 0, as_stream(stream)>>>(y, x, (float)alpha, n, lo, hi,
                                                                   i_base, nplanes);
  return launch_status("sgb_box_axpy_f32");
}

int sgb_box_axpy_f64(double* y, const double* x, double alpha, int n, int lo, int hi,
                     int i_base, int nplanes, sgb_stream_t stream) {
  if (!y || !x || n <= 0 || nplanes <= 0) return SGB_EINVAL;
  dim3 g((unsigned)((n + 255) / 256), (unsigned)((n + 3) / 4), (unsigned)nplanes);
  box_axpy_kernel<double><<<g, dim3(64, 4), 0, as_stream(stream)>>>(y, x, alpha, n, lo, hi,
                                                                    i_base, nplanes);
  return launch_status("sgb_box_axpy_f64");
}

int sgb_box_set_f32(float* y, const float* x, double alpha, int n, int lo, int hi, int i_base,
                    int nplanes, sgb_stream_t stream) {
  if (!y || !x || n <= 0 || nplanes <= 0) return SGB_EINVAL;
  dim3 g((unsigned)((n + 255) / 256), (unsigned)((n + 3) / 4), (unsigned)nplanes);
  box_set_kernel<float><<<g, dim3(64, 4), 0, as_stream(stream)>>>(y, x, (float)alpha, n, lo, hi,
                                                                  i_base, nplanes);
  return launch_status("sgb_box_set_f32");
}

int sgb_box_set_f64(double* y, const double* x, double alpha, int n, int lo, int hi, int i_base,
                    int nplanes, sgb_stream_t stream) {
  if (!y || !x || n <= 0 || nplanes <= 0) return SGB_EINVAL;
  dim3 g((unsigned)((n + 255) / 256), (unsigned)((n + 3) / 4), (unsigned)nplanes);
  box_set_kernel<double><<<g, dim3(64, 4), 0, as_stream(stream)>>>(y, x, alpha, n, lo, hi,
                                                                   i_base, nplanes);
  return launch_status("sgb_box_set_f64");
}

int sgb_smooth5_f64(const double* src, double* dst, int n, sgb_stream_t stream) {
  if (!src || !dst || n <= 0 || src == dst) return SGB_EINVAL;
  dim3 b(64, 4), g((n + 63) / 64, (n + 3) / 4);
  smooth5_kernel<<<g, b, 0, as_stream(stream)>>>(src, dst, n);
  return launch_status("sgb_smooth5_f64");
}

}  // extern "C"
