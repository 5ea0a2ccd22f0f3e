// Runtime compilation of emitted adjoint-stencil kernels:
// NVRTC -> sm_100a cubin -> cudaLibrary -> launch.
//
// The emitter (paper_1907_02818_b200/emitter.py) turns any problem the
// reference's front end differentiates (an AdjointProgram: terms, offsets,
// partials) into CUDA source for a fused, predicated gather kernel, the way
// the reference's emit_adjoint (codegen.cpp:332-382) turns it into C/OpenMP.
// This file owns the native half: compile once per source (cached by text),
// load, look up, launch.  NVRTC is dlopen'ed so the library still loads on a
// machine without it; a missing NVRTC is reported as an error, never a
// fallback.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "sgb_common.cuh"

struct sgb_jit_kernel {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kernel = nullptr;
};

namespace {

typedef int nvrtcResult_t;
struct Nvrtc {
  void* h = nullptr;
  nvrtcResult_t (*create)(void**, const char*, const char*, int, const char* const*,
                          const char* const*) = nullptr;
  nvrtcResult_t (*compile)(void*, int, const char* const*) = nullptr;
  nvrtcResult_t (*log_size)(void*, size_t*) = nullptr;
  nvrtcResult_t (*get_log)(void*, char*) = nullptr;
  nvrtcResult_t (*cubin_size)(void*, size_t*) = nullptr;
  nvrtcResult_t (*get_cubin)(void*, char*) = nullptr;
  nvrtcResult_t (*destroy)(void**) = nullptr;
};

std::mutex g_mu;
std::unordered_map<std::string, sgb_jit_kernel*> g_cache;
std::string g_log;

bool load_nvrtc(Nvrtc& n) {
  if (n.h) return true;
  const char* names[] = {"libnvrtc.so.12", "libnvrtc.so",
                         "/usr/local/cuda/lib64/libnvrtc.so.12",
                         "/usr/local/cuda/lib64/libnvrtc.so"};
  for (const char* nm : names)
    if ((n.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL))) break;
  if (!n.h) return false;
  n.create = (decltype(n.create))dlsym(n.h, "nvrtcCreateProgram");
  n.compile = (decltype(n.compile))dlsym(n.h, "nvrtcCompileProgram");
  n.log_size = (decltype(n.log_size))dlsym(n.h, "nvrtcGetProgramLogSize");
  n.get_log = (decltype(n.get_log))dlsym(n.h, "nvrtcGetProgramLog");
  n.cubin_size = (decltype(n.cubin_size))dlsym(n.h, "nvrtcGetCUBINSize");
  n.get_cubin = (decltype(n.get_cubin))dlsym(n.h, "nvrtcGetCUBIN");
  n.destroy = (decltype(n.destroy))dlsym(n.h, "nvrtcDestroyProgram");
  return n.create && n.compile && n.log_size && n.get_log && n.cubin_size && n.get_cubin &&
         n.destroy;
}

}  // namespace

extern "C" {

const char* sgb_jit_log(void) { return g_log.c_str(); }

// Compiles `source` (CUDA C++) for sm_100a and returns the __global__
// function `name` (extern "C" in the source).  Cached by (source, name).
int sgb_jit_compile(const char* source, const char* name, sgb_jit_kernel** out) {
  if (!source || !name || !out) return SGB_EINVAL;
  std::lock_guard<std::mutex> lock(g_mu);
  const std::string key = std::string(name) + '\0' + source;
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    *out = it->second;
    return 0;
  }
  static Nvrtc nv;
  if (!load_nvrtc(nv)) {
    g_log = "NVRTC (libnvrtc.so.12) not found";
    sgb::set_error(g_log);
    return SGB_EINVAL;
  }
  void* prog = nullptr;
  if (nv.create(&prog, source, "sgb_emitted.cu", 0, nullptr, nullptr) != 0) {
    sgb::set_error("nvrtcCreateProgram failed");
    return SGB_EINVAL;
  }
  // --fmad=false: every product and sum rounded separately, like the
  // reference's emitted C (gcc -O2, x86-64 baseline: no FMA contraction), so
  // emitted variants of one program (fused / per-nest) are bitwise equal
  const char* opts[] = {"-arch=sm_100a", "--std=c++17", "-default-device", "-lineinfo",
                        "--fmad=false"};
  const int rc = nv.compile(prog, 5, opts);
  size_t ls = 0;
  nv.log_size(prog, &ls);
  g_log.assign(ls, '\0');
  if (ls) nv.get_log(prog, g_log.data());
  if (rc != 0) {
    nv.destroy(&prog);
    sgb::set_error("nvrtc compile failed: " + g_log);
    return SGB_EINVAL;
  }
  size_t cs = 0;
  nv.cubin_size(prog, &cs);
  std::vector<char> cubin(cs);
  nv.get_cubin(prog, cubin.data());
  nv.destroy(&prog);
  auto* k = new sgb_jit_kernel;
  if (cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) !=
          cudaSuccess ||
      cudaLibraryGetKernel(&k->kernel, k->lib, name) != cudaSuccess) {
    sgb::set_error(std::string("loading emitted kernel failed: ") +
                   cudaGetErrorString(cudaGetLastError()));
    delete k;
    return SGB_EINVAL;
  }
  g_cache[key] = k;
  *out = k;
  return 0;
}

// Compile-only check (no GPU needed): 0 when `source` compiles for sm_100a.
int sgb_jit_check(const char* source) {
  if (!source) return SGB_EINVAL;
  std::lock_guard<std::mutex> lock(g_mu);
  static Nvrtc nv;
  if (!load_nvrtc(nv)) {
    g_log = "NVRTC (libnvrtc.so.12) not found";
    return SGB_EINVAL;
  }
  void* prog = nullptr;
  if (nv.create(&prog, source, "sgb_emitted.cu", 0, nullptr, nullptr) != 0) return SGB_EINVAL;
  const char* opts[] = {"-arch=sm_100a", "--std=c++17", "-default-device", "--fmad=false"};
  const int rc = nv.compile(prog, 4, opts);
  size_t ls = 0;
  nv.log_size(prog, &ls);
  g_log.assign(ls, '\0');
  if (ls) nv.get_log(prog, g_log.data());
  nv.destroy(&prog);
  return rc == 0 ? 0 : SGB_EINVAL;
}

// Launches an emitted kernel: args[i] points at the i-th argument value, as
// for cudaLaunchKernel.
int sgb_jit_launch(sgb_jit_kernel* k, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                   unsigned by, unsigned bz, void** args, sgb_stream_t stream) {
  return sgb_jit_launch_smem(k, gx, gy, gz, bx, by, bz, 0, args, stream);
}

// The same with `smem` bytes of dynamic shared memory (the tiled emitted
// gather's plane rings); the kernel's limit is raised on the calling device.
int sgb_jit_launch_smem(sgb_jit_kernel* k, unsigned gx, unsigned gy, unsigned gz, unsigned bx,
                        unsigned by, unsigned bz, unsigned smem, void** args,
                        sgb_stream_t stream) {
  if (!k || !args) return SGB_EINVAL;
  if (smem > 48 * 1024) {
    cudaError_t a = cudaFuncSetAttribute((const void*)k->kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (a != cudaSuccess) {
      sgb::set_error(std::string("emitted kernel smem attribute: ") + cudaGetErrorString(a));
      return -static_cast<int>(a);
    }
  }
  cudaError_t e = cudaLaunchKernel((const void*)k->kernel, dim3(gx, gy, gz), dim3(bx, by, bz),
                                   args, smem, sgb::as_stream(stream));
  sgb::g_launches.fetch_add(1, std::memory_order_relaxed);
  if (e != cudaSuccess) {
    sgb::set_error(std::string("emitted kernel launch failed: ") + cudaGetErrorString(e));
    return -static_cast<int>(e);
  }
  return 0;
}

}  // extern "C"
