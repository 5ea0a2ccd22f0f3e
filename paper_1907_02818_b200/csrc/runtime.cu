// Launcher state shared by every entry point: run-time options (read from the
// environment ONCE, then only through sgb_set_option / sgb_get_option), the
// per-device SM count, and per-(device, kernel) dynamic shared-memory
// attributes.  Everything here is thread-safe; nothing is cached per process
// that is really per device, so one process may drive several GPUs from
// several host threads.
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "sgb_common.cuh"

namespace sgb {

namespace {

struct OptionTable {
  std::array<std::atomic<long long>, kNumOpts> value{};
  std::array<std::atomic<int>, kNumOpts> set{};
};

OptionTable& table() {
  static OptionTable t;
  return t;
}

void load_env() {
  OptionTable& t = table();
  for (int o = 0; o < kNumOpts; o++) {
    const std::string key = std::string("SGB_") + kOptNames[o];
    const char* e = std::getenv(key.c_str());
    if (e && *e) {
      t.value[o].store(std::atoll(e), std::memory_order_relaxed);
      t.set[o].store(1, std::memory_order_release);
    } else {
      t.set[o].store(0, std::memory_order_release);
      t.value[o].store(0, std::memory_order_relaxed);
    }
  }
}

std::once_flag g_env_once;

OptionTable& loaded() {
  std::call_once(g_env_once, load_env);
  return table();
}

int find_opt(const char* name) {
  if (!name) return -1;
  if (std::strncmp(name, "SGB_", 4) == 0) name += 4;
  for (int o = 0; o < kNumOpts; o++)
    if (std::strcmp(name, kOptNames[o]) == 0) return o;
  return -1;
}

constexpr int kMaxDev = 64;
std::array<std::atomic<int>, kMaxDev> g_sms{};

std::mutex g_attr_mu;
std::set<std::pair<int, const void*>>& attr_done() {
  static std::set<std::pair<int, const void*>> s;
  return s;
}

}  // namespace

long long opt(Opt o, long long dflt) {
  OptionTable& t = loaded();
  if (!t.set[o].load(std::memory_order_acquire)) return dflt;
  return t.value[o].load(std::memory_order_relaxed);
}

bool opt_flag(Opt o) { return opt(o, 0) != 0; }

int num_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 148;
  int v = g_sms[dev].load(std::memory_order_relaxed);
  if (v > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
    v = 148;
  g_sms[dev].store(v, std::memory_order_relaxed);
  return v;
}

int ensure_smem(const void* fn, size_t bytes, const char* what) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) {
    std::lock_guard<std::mutex> lock(g_attr_mu);
    auto key = std::make_pair(dev, fn);
    if (attr_done().count(key)) return 0;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) attr_done().insert(key);
  }
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": setting " + std::to_string(bytes) +
              " B of dynamic shared memory failed: " + cudaGetErrorString(e));
    return -static_cast<int>(e);
  }
  return 0;
}

void* driver_entry(const char* name) {
  static std::mutex mu;
  static std::vector<std::pair<std::string, void*>> cache;
  std::lock_guard<std::mutex> lock(mu);
  for (const auto& kv : cache)
    if (kv.first == name) return kv.second;
  cudaDriverEntryPointQueryResult q;
  void* f = nullptr;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    f = nullptr;
  cache.emplace_back(name, f);
  return f;
}

}  // namespace sgb

extern "C" {

int sgb_set_option(const char* name, long long value) {
  const int o = sgb::find_opt(name);
  if (o < 0) {
    sgb::set_error(std::string("sgb_set_option: unknown option '") + (name ? name : "") + "'");
    return SGB_EINVAL;
  }
  auto& t = sgb::loaded();
  t.value[o].store(value, std::memory_order_relaxed);
  t.set[o].store(1, std::memory_order_release);
  return 0;
}

int sgb_clear_option(const char* name) {
  const int o = sgb::find_opt(name);
  if (o < 0) {
    sgb::set_error(std::string("sgb_clear_option: unknown option '") + (name ? name : "") + "'");
    return SGB_EINVAL;
  }
  sgb::loaded().set[o].store(0, std::memory_order_release);
  return 0;
}

int sgb_get_option(const char* name, long long* value, int* is_set) {
  const int o = sgb::find_opt(name);
  if (o < 0) {
    sgb::set_error(std::string("sgb_get_option: unknown option '") + (name ? name : "") + "'");
    return SGB_EINVAL;
  }
  auto& t = sgb::loaded();
  if (is_set) *is_set = t.set[o].load(std::memory_order_acquire);
  if (value) *value = t.value[o].load(std::memory_order_relaxed);
  return 0;
}

const char* sgb_option_name(int index) {
  return index >= 0 && index < sgb::kNumOpts ? sgb::kOptNames[index] : nullptr;
}

}  // extern "C"
