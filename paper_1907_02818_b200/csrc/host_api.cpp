// C++ host API (include/stencilgrad_b200.hpp): the reference's interp.hpp
// entry points (run_nest / run_program / run_scatter_adjoint,
// interp.hpp:45-103) over the C ABI.  Upload every referenced grid, launch the
// sm_100a kernel through the C entry, download the written grids into a copy
// of the Env.  No CPU compute path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>
#include <sstream>
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

// ---------------------------------------------------------------- verification
// The reference's verification entry points (interp.cpp:232-435) over the
// B200 kernels.  The draws, steps and thresholds follow the reference so a
// report can be read beside its own; every stencil evaluation (primal, gather
// adjoint, scatter adjoint) is a kernel launch through the C ABI.
namespace {

bool has_adjoint(const Family& f, const std::string& array) {
  return std::find(f.adjoint.begin(), f.adjoint.end(), array + "_b") != f.adjoint.end();
}

// active inputs (declaration order), i.e. active arrays other than the output
std::vector<std::string> active_inputs(const Family& f) {
  std::vector<std::string> in;
  for (const auto& a : f.primal)
    if (a != f.out && has_adjoint(f, a)) in.push_back(a);
  return in;
}

void fill_normal(DenseGrid& g, std::mt19937_64& rng) {  // interp.cpp:242-245
  std::normal_distribution<double> nd(0.0, 1.0);
  for (double& x : g.data()) x = nd(rng);
}

std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b) {  // :232-240
  std::uint64_t x = seed + 0x9E3779B97F4A7C15ull * (a + 1) + 0xBF58476D1CE4E5B9ull * (b + 1);
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

// tie_gap_of (interp.cpp:255-263): the smallest |a - b| over the min/max nodes
// of the primal body on its iteration space.  Only burgers2d has such nodes
// (max(u_1, 0), min(u_1, 0) at the centre point): min |u_1| over [1, n-2]^2.
double tie_gap_of(const Family& f, const Env& env) {
  double gap = std::numeric_limits<double>::infinity();
  if (std::string(f.name) != "burgers2d") return gap;
  const long long n = env.sizes.at("n");
  const std::vector<double>& u = env.grids.at("u_1").data();
  for (long long i = 1; i <= n - 2; i++)
    for (long long j = 1; j <= n - 2; j++) gap = std::min(gap, std::fabs(u[i * n + j]));
  return gap;
}

std::string shortest(double v) {  // shortest decimal that round-trips (JSON numbers)
  char buf[40];
  for (int p = 1; p <= 17; p++) {
    std::snprintf(buf, sizeof(buf), "%.*g", p, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  return buf;
}

}  // namespace

Env make_env(const std::string& family, const std::map<std::string, long long>& sizes,
             std::uint64_t seed) {
  const Family& f = find_family(family);
  const auto nit = sizes.find("n");
  if (nit == sizes.end()) throw Error("size symbol 'n' missing");
  const std::vector<long long> shape(f.d, nit->second);
  Env env;
  env.sizes = sizes;
  env.seed = seed;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> nd(0.0, 1.0);
  for (const auto& s : f.scalars) env.scalars[s] = nd(rng);
  for (const auto& a : f.primal) {
    DenseGrid g(shape);
    fill_normal(g, rng);
    env.grids[a] = std::move(g);
  }
  for (const auto& a : f.primal) {
    if (!has_adjoint(f, a)) continue;
    DenseGrid g(shape);
    if (a == f.out) fill_normal(g, rng);
    env.grids[a + "_b"] = std::move(g);
  }
  return env;
}

GridCompare compare_grids(const DenseGrid& a, const DenseGrid& b, double rel_tol) {
  if (a.shape() != b.shape()) throw Error("grid shape mismatch");
  const std::size_t count = a.data().size();
  if (count == 0) return {0.0, 0.0 <= rel_tol};
  DeviceGrids<double> dev;
  for (const DenseGrid* g : {&a, &b}) {
    double* d = nullptr;
    cuda_check(cudaMalloc(&d, count * sizeof(double)), "cudaMalloc");
    dev.p.push_back(d);
    cuda_check(cudaMemcpy(d, g->data().data(), count * sizeof(double), cudaMemcpyHostToDevice),
               "H2D");
  }
  double out4[4] = {0, 0, 0, 0};
  if (sgb_compare_f64(dev.p[0], dev.p[1], (long long)count, out4, nullptr) != 0)
    throw Error(std::string("compare_grids: ") + sgb_last_error());
  return {out4[0], out4[0] <= rel_tol};
}

DotReport dot_product_test(const std::string& family, const Env& env, int trials) {
  if (trials < 1) throw Error("dot-product test needs at least one trial");
  const Family& f = find_family(family);
  const double threshold = 1e-4;  // every family is nonlinear in its active inputs
  const std::vector<std::string> inputs = active_inputs(f);
  const bool piecewise = std::string(f.name) == "burgers2d";
  double max_err = 0.0;
  for (int t = 0; t < trials; t++) {
    for (std::uint64_t attempt = 0;; attempt++) {
      if (attempt > 200) throw Error("no tie-free base point found after 200 redraws");
      std::mt19937_64 rng(mix_seed(env.seed, static_cast<std::uint64_t>(t), attempt));
      Env base = env;
      if (attempt > 0)
        for (const auto& a : inputs) fill_normal(base.grids.at(a), rng);
      if (piecewise && tie_gap_of(f, base) < 1e-3) continue;

      std::map<std::string, DenseGrid> v;
      for (const auto& a : inputs) {
        DenseGrid g(base.grids.at(a).shape());
        fill_normal(g, rng);
        v[a] = std::move(g);
      }
      DenseGrid w(base.grids.at(f.out).shape());
      fill_normal(w, rng);

      double umax = 0.0;
      for (const auto& a : inputs)
        for (double x : base.grids.at(a).data()) umax = std::max(umax, std::fabs(x));
      const double h = 1e-5 * (1.0 + umax);

      Env plus = base, minus = base;
      for (const auto& a : inputs) {
        auto& gp = plus.grids.at(a).data();
        auto& gm = minus.grids.at(a).data();
        const auto& gv = v.at(a).data();
        for (std::size_t i = 0; i < gv.size(); i++) {
          gp[i] += h * gv[i];
          gm[i] -= h * gv[i];
        }
      }
      const Env rp = run_nest(family, plus);   // primal kernel
      const Env rm = run_nest(family, minus);
      double lhs = 0.0;
      {
        const auto& dp = rp.grids.at(f.out).data();
        const auto& dm = rm.grids.at(f.out).data();
        for (std::size_t i = 0; i < dp.size(); i++)
          lhs += w.data()[i] * (dp[i] - dm[i]) / (2.0 * h);
      }

      Env aenv = base;
      aenv.grids.at(f.seed) = w;
      for (const auto& a : inputs) {
        auto& g = aenv.grids.at(a + "_b");
        std::fill(g.data().begin(), g.data().end(), 0.0);
      }
      const Env res = run_program(family, aenv);  // gather adjoint kernel
      double rhs = 0.0;
      for (const auto& a : inputs) {
        const auto& gu = res.grids.at(a + "_b").data();
        const auto& gv = v.at(a).data();
        for (std::size_t i = 0; i < gu.size(); i++) rhs += gv[i] * gu[i];
      }
      max_err = std::max(max_err, std::fabs(lhs - rhs) / (1.0 + std::fabs(rhs)));
      break;
    }
  }
  return {max_err, threshold, trials, max_err <= threshold};
}

bool VerifyReport::pass() const {
  return std::all_of(checks.begin(), checks.end(), [](const CheckLine& c) { return c.pass; });
}

std::string VerifyReport::text() const {
  std::ostringstream os;
  for (const auto& c : checks) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "%-20s max_rel_err=%.6e threshold=%.1e %s", c.name.c_str(),
                  c.metric, c.threshold, c.pass ? "PASS" : "FAIL");
    os << buf << "\n";
  }
  return os.str();
}

std::string VerifyReport::json_text() const {
  std::ostringstream os;
  os << "{\n  \"checks\": [";
  for (std::size_t i = 0; i < checks.size(); i++) {
    const CheckLine& c = checks[i];
    os << (i ? "," : "") << "\n    {\n      \"name\": \"" << c.name << "\",\n      \"metric\": "
       << shortest(c.metric) << ",\n      \"threshold\": " << shortest(c.threshold)
       << ",\n      \"pass\": " << (c.pass ? "true" : "false") << "\n    }";
  }
  os << (checks.empty() ? "]" : "\n  ]") << ",\n  \"pass\": " << (pass() ? "true" : "false")
     << "\n}\n";
  return os.str();
}

VerifyReport verify_problem(const std::string& family,
                            const std::map<std::string, long long>& sizes, std::uint64_t seed,
                            int trials, bool fd) {
  const Family& f = find_family(family);
  VerifyReport report;
  const Env env = make_env(family, sizes, seed);
  const Env gather = run_program(family, env);
  const Env scatter = run_scatter_adjoint(family, env);
  double metric = 0.0;
  for (const auto& a : active_inputs(f)) {
    const GridCompare c = compare_grids(gather.grids.at(a + "_b"), scatter.grids.at(a + "_b"),
                                        1e-12);
    metric = std::max(metric, c.max_rel_err);
  }
  report.checks.push_back({"oracle-equivalence", metric, 1e-12, metric <= 1e-12});
  if (fd) {
    const DotReport d = dot_product_test(family, env, trials);
    report.checks.push_back({"dot-product", d.max_rel_err, d.threshold, d.pass});
  }
  return report;
}

std::vector<std::string> array_params(const std::string& family, const std::string& kind) {
  const Family& f = find_family(family);
  if (kind == "primal") return f.primal;
  if (kind == "adjoint" || kind == "scatter") return f.adjoint;
  throw Error("kind must be primal, adjoint or scatter");
}

}  // namespace sgb
