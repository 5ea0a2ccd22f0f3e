// Device-side parity reductions: the reference's compare_grids metric
// (interp.cpp:290-298: max_i |a - b| / (1 + |b|)) and the dot products of its
// dot_product_test (interp.cpp:354-375), evaluated in fp64 on the B200 so a
// full-size check (1024^3: 8.6 GB per fp64 grid) never downloads the kernel's
// output.  Verification entries: synchronous, deterministic (per-block partials
// reduced in a fixed order by one CTA).
#include <cuda_runtime.h>

#include <cmath>
#include <string>

#include "sgb_common.cuh"

namespace sgb {

constexpr int kVerifyThreads = 256;
constexpr int kVerifyBlocks = 148 * 4;

// out per block: [max rel err, sum (a-b)^2, sum b^2, non-finite count]
template <typename T>
__global__ void __launch_bounds__(kVerifyThreads)
    compare_partial_kernel(const T* __restrict__ a, const double* __restrict__ b,
                           long long count, double* __restrict__ part) {
  double mx = 0.0, se = 0.0, sb = 0.0, bad = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const double x = (double)a[i], y = b[i];
    const double d = x - y;
    const double r = fabs(d) / (1.0 + fabs(y));
    if (!isfinite(r)) {
      bad += 1.0;
    } else {
      mx = fmax(mx, r);
      se = fma(d, d, se);
      sb = fma(y, y, sb);
    }
  }
  __shared__ double sh[4][kVerifyThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    se += __shfl_xor_sync(0xffffffffu, se, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
  }
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  if (l == 0) {
    sh[0][w] = mx;
    sh[1][w] = se;
    sh[2][w] = sb;
    sh[3][w] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kVerifyThreads / 32; ++k) {
      mx = fmax(mx, sh[0][k]);
      se += sh[1][k];
      sb += sh[2][k];
      bad += sh[3][k];
    }
    double* p = part + 4 * blockIdx.x;
    p[0] = mx;
    p[1] = se;
    p[2] = sb;
    p[3] = bad;
  }
}

template <typename T>
__global__ void __launch_bounds__(kVerifyThreads)
    dot_partial_kernel(const T* __restrict__ a, const T* __restrict__ b, long long count,
                       double* __restrict__ part) {
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
    s = fma((double)a[i], (double)b[i], s);
  __shared__ double sh[kVerifyThreads / 32];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x % 32 == 0) sh[threadIdx.x / 32] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < kVerifyThreads / 32; ++k) s += sh[k];
    part[4 * blockIdx.x] = s;
  }
}

// fixed-order final reduction of the per-block partials (one thread: <= 592
// entries, deterministic)
__global__ void finish_kernel(const double* __restrict__ part, int nblocks, int mode,
                              double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mx = 0.0, se = 0.0, sb = 0.0, bad = 0.0;
  for (int k = 0; k < nblocks; ++k) {
    const double* p = part + 4 * k;
    if (mode == 0) {
      mx = fmax(mx, p[0]);
      se += p[1];
      sb += p[2];
      bad += p[3];
    } else {
      se += p[0];
    }
  }
  out[0] = mx;
  out[1] = se;
  out[2] = sb;
  out[3] = bad;
}

template <typename Launch>
static int reduce_call(const char* name, long long count, double* out4, cudaStream_t s, int mode,
                       Launch launch) {
  if (count < 0 || !out4) {
    set_error(std::string(name) + ": bad arguments");
    return SGB_EINVAL;
  }
  long long blocks = (count + kVerifyThreads - 1) / kVerifyThreads;
  const int nb = (int)(blocks < 1 ? 1 : blocks > kVerifyBlocks ? kVerifyBlocks : blocks);
  double* part = nullptr;
  cudaError_t e = cudaMallocAsync(&part, sizeof(double) * (4 * nb + 4), s);
  if (e != cudaSuccess) {
    set_error(std::string(name) + ": " + cudaGetErrorString(e));
    return -(int)e;
  }
  launch(nb, part);
  int rc = launch_status(name);
  if (rc == 0) {
    finish_kernel<<<1, 32, 0, s>>>(part, nb, mode, part + 4 * nb);
    rc = launch_status(name);
  }
  if (rc == 0) {
    e = cudaMemcpyAsync(out4, part + 4 * nb, 4 * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
      set_error(std::string(name) + ": " + cudaGetErrorString(e));
      rc = -(int)e;
    }
  }
  cudaFreeAsync(part, s);
  return rc;
}

template <typename T>
static int compare(const char* name, const T* a, const double* b, long long count, double* out4,
                   cudaStream_t s) {
  if (count > 0 && (!a || !b)) {
    set_error(std::string(name) + ": null array");
    return SGB_EINVAL;
  }
  return reduce_call(name, count, out4, s, 0, [&](int nb, double* part) {
    compare_partial_kernel<T><<<nb, kVerifyThreads, 0, s>>>(a, b, count, part);
  });
}

template <typename T>
static int dot(const char* name, const T* a, const T* b, long long count, double* out,
               cudaStream_t s) {
  if (count > 0 && (!a || !b)) {
    set_error(std::string(name) + ": null array");
    return SGB_EINVAL;
  }
  double o4[4];
  const int rc = reduce_call(name, count, o4, s, 1, [&](int nb, double* part) {
    dot_partial_kernel<T><<<nb, kVerifyThreads, 0, s>>>(a, b, count, part);
  });
  if (rc == 0 && out) *out = o4[1];
  return rc;
}

}  // namespace sgb

extern "C" {

int sgb_compare_f32(const float* a, const double* b, long long count, double* out4,
                    sgb_stream_t stream) {
  return sgb::compare("sgb_compare_f32", a, b, count, out4, sgb::as_stream(stream));
}
int sgb_compare_f64(const double* a, const double* b, long long count, double* out4,
                    sgb_stream_t stream) {
  return sgb::compare("sgb_compare_f64", a, b, count, out4, sgb::as_stream(stream));
}
int sgb_dot_f32(const float* a, const float* b, long long count, double* out,
                sgb_stream_t stream) {
  return sgb::dot("sgb_dot_f32", a, b, count, out, sgb::as_stream(stream));
}
int sgb_dot_f64(const double* a, const double* b, long long count, double* out,
                sgb_stream_t stream) {
  return sgb::dot("sgb_dot_f64", a, b, count, out, sgb::as_stream(stream));
}

}  // extern "C"
