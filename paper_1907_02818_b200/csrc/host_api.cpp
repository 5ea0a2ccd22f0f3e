// C++ host API (include/stencilgrad_b200.hpp): the reference's interp.hpp
// entry points (run_nest / run_program / run_scatter_adjoint,
// interp.hpp:45-103) over the C ABI.  Upload every referenced grid, launch the
// sm_100a kernel through the C entry, download the written grids into a copy
// of the Env.  No CPU compute path.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "stencilgrad_b200.h"
#include "stencilgrad_b200.hpp"

namespace sgb {

DenseGrid::DenseGrid(std::vector<long long> shape) : shape_(std::move(shape)) {
  std::size_t total = 1;
  for (long long e : shape_) {
    if (e < 0) throw Error("DenseGrid: negative extent");
    total *= static_cast<std::size_t>(e);
  }
  data_.assign(total, 0.0);
}

bool DenseGrid::in_bounds(const std::vector<long long>& idx) const {
  if (idx.size() != shape_.size()) return false;
  for (std::size_t d = 0; d < idx.size(); d++)
    if (idx[d] < 0 || idx[d] >= shape_[d]) return false;
  return true;
}

std::size_t DenseGrid::flat(const std::vector<long long>& idx) const {
  if (!in_bounds(idx)) throw Error("DenseGrid: index out of bounds");
  std::size_t f = 0;
  for (std::size_t d = 0; d < idx.size(); d++) f = f * shape_[d] + idx[d];
  return f;
}

namespace {

// The five families' spec-level facts (oracle/specs/<family>.json; array
// order = the reference emitter's parameter order, codegen.cpp:198-230).
struct Family {
  const char* name;
  int d;
  std::vector<std::string> scalars, primal, adjoint;
  std::string out, seed;
};

const std::vector<Family>& families() {
  static const std::vector<Family> f = {
      {"wave1d", 1, {"D"}, {"c", "u", "u_prev", "u_next"},
       {"c", "c_b", "u", "u_b", "u_prev_b", "u_next_b"}, "u_next", "u_next_b"},
      {"wave3d_c", 3, {"D"}, {"c", "u_1", "u_2", "u"},
       {"c", "c_b", "u_1", "u_1_b", "u_2_b", "u_b"}, "u", "u_b"},
      {"wave3d_c2", 3, {"D"}, {"c", "u_1", "u_2", "u"},
       {"c", "c_b", "u_1", "u_1_b", "u_2_b", "u_b"}, "u", "u_b"},
      {"burgers2d", 2, {"C", "D"}, {"u_1", "u"}, {"u_1", "u_1_b", "u_b"}, "u", "u_b"},
      {"wave3d_r4", 3, {"D"}, {"c", "u_1", "u_2", "u"}, {"c", "c_b", "u_1", "u_1_b", "u_b"},
       "u", "u_b"},
  };
  return f;
}

const Family& find_family(const std::string& name) {
  for (const auto& f : families())
    if (name == f.name) return f;
  throw Error("unsupported problem '" + name +
              "' (wave1d, wave3d_c, wave3d_c2, burgers2d, wave3d_r4)");
}

#define SGB_DISPATCH_WAVE(NAME, SFX)                                                          \
  if (fam == #NAME) {                                                                         \
    if (kind == 0) return NAME##_##SFX(n, sc[0], a[0], a[1], a[2], a[3], nullptr);            \
    if (kind == 1) return NAME##_b_##SFX(n, sc[0], a[0], a[1], a[2], a[3], a[4], a[5], nullptr); \
    return NAME##_scatter_b_##SFX(n, sc[0], a[0], a[1], a[2], a[3], a[4], a[5], nullptr);     \
  }

template <typename T>
int launch(const std::string& fam, int kind, int n, const double* sc, T** a);

template <>
int launch<double>(const std::string& fam, int kind, int n, const double* sc, double** a) {
  SGB_DISPATCH_WAVE(wave1d, f64)
  SGB_DISPATCH_WAVE(wave3d_c, f64)
  SGB_DISPATCH_WAVE(wave3d_c2, f64)
  if (fam == "burgers2d") {
    if (kind == 0) return burgers2d_f64(n, sc[0], sc[1], a[0], a[1], nullptr);
    if (kind == 1) return burgers2d_b_f64(n, sc[0], sc[1], a[0], a[1], a[2], nullptr);
    return burgers2d_scatter_b_f64(n, sc[0], sc[1], a[0], a[1], a[2], nullptr);
  }
  if (kind == 0) return wave3d_r4_f64(n, sc[0], a[0], a[1], a[2], a[3], nullptr);
  if (kind == 1) return wave3d_r4_b_f64(n, sc[0], a[0], a[1], a[2], a[3], a[4], nullptr);
  return wave3d_r4_scatter_b_f64(n, sc[0], a[0], a[1], a[2], a[3], a[4], nullptr);
}

template <>
int launch<float>(const std::string& fam, int kind, int n, const double* sc, float** a) {
  SGB_DISPATCH_WAVE(wave1d, f32)
  SGB_DISPATCH_WAVE(wave3d_c, f32)
  SGB_DISPATCH_WAVE(wave3d_c2, f32)
  if (fam == "burgers2d") {
    if (kind == 0) return burgers2d_f32(n, sc[0], sc[1], a[0], a[1], nullptr);
    if (kind == 1) return burgers2d_b_f32(n, sc[0], sc[1], a[0], a[1], a[2], nullptr);
    return burgers2d_scatter_b_f32(n, sc[0], sc[1], a[0], a[1], a[2], nullptr);
  }
  if (kind == 0) return wave3d_r4_f32(n, sc[0], a[0], a[1], a[2], a[3], nullptr);
  if (kind == 1) return wave3d_r4_b_f32(n, sc[0], a[0], a[1], a[2], a[3], a[4], nullptr);
  return wave3d_r4_scatter_b_f32(n, sc[0], a[0], a[1], a[2], a[3], a[4], nullptr);
}
#undef SGB_DISPATCH_WAVE

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename T>
struct DeviceGrids {
  std::vector<T*> p;
  ~DeviceGrids() {
    for (T* q : p) cudaFree(q);
  }
};

// kind: 0 primal, 1 gather adjoint, 2 scatter adjoint
template <typename T>
Env run(const std::string& family, const Env& env, int kind) {
  const Family& f = find_family(family);
  const auto nit = env.sizes.find("n");
  if (nit == env.sizes.end()) throw Error("size symbol 'n' missing from Env");
  const long long n = nit->second;
  if (n <= 0 || n > (1LL << 31) - 1) throw Error("size n out of range");
  std::vector<long long> shape(f.d, n);
  std::size_t count = 1;
  for (int d = 0; d < f.d; d++) count *= static_cast<std::size_t>(n);
  double sc[2] = {0.0, 0.0};
  for (std::size_t s = 0; s < f.scalars.size(); s++) {
    const auto it = env.scalars.find(f.scalars[s]);
    if (it == env.scalars.end()) throw Error("scalar '" + f.scalars[s] + "' missing from Env");
    sc[s] = it->second;
  }
  const std::vector<std::string>& names = kind == 0 ? f.primal : f.adjoint;
  DeviceGrids<T> dev;
  std::vector<T> stage(count);
  for (const auto& nm : names) {
    const auto it = env.grids.find(nm);
    if (it == env.grids.end()) throw Error("grid '" + nm + "' missing from Env");
    if (it->second.shape() != shape) throw Error("grid '" + nm + "' has the wrong shape");
    T* d = nullptr;
    cuda_check(cudaMalloc(&d, count * sizeof(T)), "cudaMalloc");
    dev.p.push_back(d);
    const std::vector<double>& h = it->second.data();
    if (std::is_same<T, double>::value) {
      cuda_check(cudaMemcpy(d, h.data(), count * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    } else {
      std::transform(h.begin(), h.end(), stage.begin(), [](double v) { return (T)v; });
      cuda_check(cudaMemcpy(d, stage.data(), count * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
  }
  const int rc = launch<T>(family, kind, (int)n, sc, dev.p.data());
  if (rc == 1) throw Error("minimum extent guard violated (adjoint.cpp:134-143)");
  if (rc != 0) throw Error(std::string("B200 kernel failed: ") + sgb_last_error());
  cuda_check(cudaDeviceSynchronize(), "kernel");
  Env out = env;
  for (std::size_t a = 0; a < names.size(); a++) {
    const std::string& nm = names[a];
    const bool written = kind == 0 ? nm == f.out
                                   : (nm.size() > 2 && nm.compare(nm.size() - 2, 2, "_b") == 0 &&
                                      nm != f.seed);
    if (!written) continue;
    std::vector<double>& h = out.grids[nm].data();
    if (std::is_same<T, double>::value) {
      cuda_check(cudaMemcpy(h.data(), dev.p[a], count * sizeof(T), cudaMemcpyDeviceToHost),
                 "D2H");
    } else {
      cuda_check(cudaMemcpy(stage.data(), dev.p[a], count * sizeof(T), cudaMemcpyDeviceToHost),
                 "D2H");
      std::transform(stage.begin(), stage.end(), h.begin(), [](T v) { return (double)v; });
    }
  }
  return out;
}

Env dispatch(const std::string& family, const Env& env, Precision p, int kind) {
  return p == Precision::f64 ? run<double>(family, env, kind) : run<float>(family, env, kind);
}

}  // namespace

Env run_nest(const std::string& family, const Env& env, Precision p) {
  return dispatch(family, env, p, 0);
}
Env run_program(const std::string& family, const Env& env, Precision p) {
  return dispatch(family, env, p, 1);
}
Env run_scatter_adjoint(const std::string& family, const Env& env, Precision p) {
  return dispatch(family, env, p, 2);
}

Program Program::of(const std::string& family) {
  const char* t = sgb_program_text(family.c_str());
  if (!t) throw Error(sgb_last_error());
  return Program{t};
}

std::string Program::family() const {
  const char* f = sgb_program_family(text.c_str());
  if (!f) throw Error(std::string("no B200 kernel computes this program: ") + sgb_last_error());
  return f;
}

Env run_program(const Program& program, const Env& env, Precision p) {
  return dispatch(program.family(), env, p, 1);
}

std::vector<std::string> array_params(const std::string& family, const std::string& kind) {
  const Family& f = find_family(family);
  if (kind == "primal") return f.primal;
  if (kind == "adjoint" || kind == "scatter") return f.adjoint;
  throw Error("kind must be primal, adjoint or scatter");
}

}  // namespace sgb
