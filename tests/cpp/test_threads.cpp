// Host-thread safety of the C ABI: the launchers' per-
// device state (dynamic shared-memory attributes, SM counts, tensor-map
// encoder, side streams) is initialised once per device under std::call_once
// / mutexes, so T host threads that make their FIRST calls at the same
// moment -- each on its own stream and buffers -- must all succeed and
// produce bitwise the result of one serial call.  Covers the fp32 radius-4
// (v7, split / forked launches), radius-1 (v1) and fp64 radius-4 streaming
// kernels and the fused-fresh form, on every visible device (the 8-GPU box:
// devices 0..7 from one process).  Built and run by tests/test_threads.py.
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "stencilgrad_b200.h"

#define CUDA_OK(x)                                                                  \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      std::fprintf(stderr, "%s:%d: %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(2);                                                                 \
    }                                                                               \
  } while (0)

enum Kind { R4_F32, R4_FRESH_F32, C_F32, R4_F64 };
static const char* kName[] = {"wave3d_r4_b_f32", "wave3d_r4_b_fresh_f32", "wave3d_c_b_f32",
                              "wave3d_r4_b_f64"};

struct Job {
  Kind kind;
  int n;
  size_t elem;
  std::vector<void*> a;  // c, c_b, u_1, u_1_b, u_b, (u_2_b)
};

static Job make_job(Kind kind, int n, unsigned seed) {
  Job j{kind, n, kind == R4_F64 ? sizeof(double) : sizeof(float), {}};
  const int arrays = kind == C_F32 ? 6 : 5;
  const size_t bytes = (size_t)n * n * n * j.elem;
  for (int k = 0; k < arrays; k++) {
    void* p = nullptr;
    CUDA_OK(cudaMalloc(&p, bytes));
    int rc = j.elem == 4 ? sgb_fill_normal3d_f32((float*)p, n, 0, n, 0, seed, 10 + k, k == 0 ? 3.0 : 0.0,
                                                 k == 0 ? 0.5 : 1.0, nullptr)
                         : sgb_fill_normal3d_f64((double*)p, n, 0, n, 0, seed, 10 + k,
                                                 k == 0 ? 3.0 : 0.0, k == 0 ? 0.5 : 1.0, nullptr);
    if (rc) {
      std::fprintf(stderr, "fill: %s\n", sgb_last_error());
      std::exit(2);
    }
    j.a.push_back(p);
  }
  CUDA_OK(cudaDeviceSynchronize());
  return j;
}

static Job clone(const Job& src) {
  Job j{src.kind, src.n, src.elem, {}};
  const size_t bytes = (size_t)src.n * src.n * src.n * src.elem;
  for (void* s : src.a) {
    void* p = nullptr;
    CUDA_OK(cudaMalloc(&p, bytes));
    CUDA_OK(cudaMemcpy(p, s, bytes, cudaMemcpyDeviceToDevice));
    j.a.push_back(p);
  }
  return j;
}

static int run(const Job& j, cudaStream_t s) {
  auto f = [&](int k) { return (float*)j.a[k]; };
  auto d = [&](int k) { return (double*)j.a[k]; };
  switch (j.kind) {
    case R4_F32: return wave3d_r4_b_f32(j.n, 0.01, f(0), f(1), f(2), f(3), f(4), s);
    case R4_FRESH_F32: return wave3d_r4_b_fresh_f32(j.n, 0.01, f(0), f(1), f(2), f(3), f(4), s);
    case C_F32: return wave3d_c_b_f32(j.n, 0.1, f(0), f(1), f(2), f(3), f(5), f(4), s);
    case R4_F64: return wave3d_r4_b_f64(j.n, 0.01, d(0), d(1), d(2), d(3), d(4), s);
  }
  return -1;
}

static std::vector<char> outputs(const Job& j) {
  const size_t bytes = (size_t)j.n * j.n * j.n * j.elem;
  std::vector<char> h;
  for (int k : {1, 3, 5}) {
    if (k >= (int)j.a.size()) continue;
    std::vector<char> b(bytes);
    CUDA_OK(cudaMemcpy(b.data(), j.a[k], bytes, cudaMemcpyDeviceToHost));
    h.insert(h.end(), b.begin(), b.end());
  }
  return h;
}

int main(int argc, char** argv) {
  const int threads = argc > 1 ? std::atoi(argv[1]) : 8;
  const int iters = argc > 2 ? std::atoi(argv[2]) : 3;
  int devices = 0;
  CUDA_OK(cudaGetDeviceCount(&devices));
  int failures = 0, checks = 0;
  // per device: T jobs (kinds round-robin), each thread owns one; the serial
  // reference runs in the SAME process only after the threaded runs, so the
  // threads are the first callers on every device
  struct Dev {
    std::vector<Job> jobs, refs;
  };
  std::vector<Dev> dev(devices);
  const Kind kinds[] = {R4_F32, R4_FRESH_F32, C_F32, R4_F64};
  const int sizes[] = {72, 68, 64, 40};
  for (int d = 0; d < devices; d++) {
    CUDA_OK(cudaSetDevice(d));
    for (int t = 0; t < threads; t++) {
      const Kind k = kinds[t % 4];
      dev[d].jobs.push_back(make_job(k, sizes[t % 4], 100 + t));
      dev[d].refs.push_back(clone(dev[d].jobs.back()));
    }
  }
  std::mutex mu;
  std::condition_variable cv;
  bool go = false;
  std::atomic<int> errors{0};
  std::vector<std::thread> pool;
  for (int d = 0; d < devices; d++)
    for (int t = 0; t < threads; t++)
      pool.emplace_back([&, d, t] {
        CUDA_OK(cudaSetDevice(d));
        cudaStream_t s;
        CUDA_OK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return go; });
        }
        for (int it = 0; it < iters; it++)
          if (int rc = run(dev[d].jobs[t], s)) {
            std::fprintf(stderr, "device %d thread %d %s: rc %d (%s)\n", d, t,
                         kName[dev[d].jobs[t].kind], rc, sgb_last_error());
            errors++;
          }
        CUDA_OK(cudaStreamSynchronize(s));
        CUDA_OK(cudaStreamDestroy(s));
      });
  {
    std::lock_guard<std::mutex> lk(mu);
    go = true;
  }
  cv.notify_all();
  for (auto& th : pool) th.join();
  failures += errors.load();
  for (int d = 0; d < devices; d++) {
    CUDA_OK(cudaSetDevice(d));
    for (int t = 0; t < threads; t++) {
      for (int it = 0; it < iters; it++)
        if (run(dev[d].refs[t], nullptr)) failures++;
      CUDA_OK(cudaDeviceSynchronize());
      checks++;
      if (outputs(dev[d].jobs[t]) != outputs(dev[d].refs[t])) {
        std::fprintf(stderr, "device %d thread %d %s: differs from the serial call\n", d, t,
                     kName[dev[d].jobs[t].kind]);
        failures++;
      }
    }
  }
  std::printf("devices %d threads %d iters %d: %d checks, %d failures\n", devices, threads,
              iters, checks, failures);
  return failures ? 1 : 0;
}
