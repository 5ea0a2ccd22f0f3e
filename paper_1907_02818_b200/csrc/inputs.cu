// Device-side synthetic input generation (BASELINE.json distributions).
//
// Counter-based: every value is a pure function of (seed, stream_id, global
// flat index), so slabs of any z-decomposition regenerate exactly the values
// a single GPU would hold -- the property the multi-GPU runs rely on to be
// compared against one oracle output.
#include "sgb_common.cuh"

namespace sgb {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

__device__ __forceinline__ uint64_t hash3(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return mix64(seed * 0x9E3779B97F4A7C15ull + mix64(stream + 0xD1B54A32D192ED03ull) + ctr);
}

// kind 0: N(mean, scale^2) by Box-Muller in fp64; kind 1: U[mean, mean + scale)
__device__ __forceinline__ double draw(uint64_t seed, uint64_t stream, uint64_t idx, int kind) {
  const uint64_t h1 = hash3(seed, stream, 2 * idx), h2 = hash3(seed, stream, 2 * idx + 1);
  const double u2 = (double)(h2 >> 11) * 0x1.0p-53;
  if (kind == 1) return u2;
  const double u1 = (double)((h1 >> 11) + 1) * 0x1.0p-53;  // (0, 1]
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
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

int sgb_fill_layered_f32(float* c, int n, int layers, double lo, double hi, uint64_t seed,
                         int i_base, int nplanes, sgb_stream_t stream) {
  if (!c || n <= 0 || layers <= 0 || nplanes <= 0) return SGB_EINVAL;
  layered_kernel<<<fill_grid((long long)nplanes * n * n), 256, 0, as_stream(stream)>>>(
      c, n, layers, lo, hi, seed, i_base, nplanes);
  return launch_status("sgb_fill_layered_f32");
}

int sgb_smooth5_f64(const double* src, double* dst, int n, sgb_stream_t stream) {
  if (!src || !dst || n <= 0 || src == dst) return SGB_EINVAL;
  dim3 b(64, 4), g((n + 63) / 64, (n + 3) / 4);
  smooth5_kernel<<<g, b, 0, as_stream(stream)>>>(src, dst, n);
  return launch_status("sgb_smooth5_f64");
}

}  // extern "C"
