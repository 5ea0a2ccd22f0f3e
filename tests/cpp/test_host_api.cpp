// C++ host API parity test (include/stencilgrad_b200.hpp), written like the
// reference's own interp tests (proj/tests/test_interp.cpp: run_program /
// run_nest / run_scatter_adjoint on an Env, compare_grids at 1e-12, guard
// violations throw).  The checker is the repo's C oracle (oracle/sg_oracle.c,
// pinned to the reference by tests/test_oracle_pins.py) -- test
// infrastructure, linked only here.  Needs a GPU; built and run by
// tests/test_host_api.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>

#include "sg_oracle.h"
#include "stencilgrad_b200.hpp"

static int g_checks = 0, g_failures = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    g_checks++;                                                                  \
    if (!(cond)) {                                                               \
      g_failures++;                                                              \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                            \
  } while (0)

static double compare(const sgb::DenseGrid& a, const std::vector<double>& b) {
  double e = 0;  // compare_grids (interp.cpp:290-298)
  for (std::size_t i = 0; i < b.size(); i++)
    e = std::fmax(e, std::fabs(a.data()[i] - b[i]) / (1 + std::fabs(b[i])));
  return e;
}

// Env with every array and adjoint of the family (oracle declaration order),
// seeded: c ~ U[1.5, 4.5], Burgers u ~ U[-1, 1], the rest N(0, 1).
static sgb::Env make_env(int fam, long long n, unsigned seed) {
  const sg_family* f = sg_family_get(fam);
  sgb::Env env;
  env.sizes["n"] = n;
  for (int s = 0; s < f->nscalars; s++) env.scalars[f->scalars[s]] = 0.1 + 0.05 * s;
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> N(0.0, 1.0);
  std::uniform_real_distribution<double> U(1.5, 4.5), V(-1.0, 1.0);
  std::vector<long long> shape(f->d, n + f->shape_n);
  for (int a = 0; a < f->narrays; a++) {
    sgb::DenseGrid g(shape), b(shape);
    const std::string nm = f->arrays[a];
    for (double& v : g.data()) v = nm == "c" ? U(rng) : (fam == SG_BURGERS2D ? V(rng) : N(rng));
    for (double& v : b.data()) v = N(rng);
    env.grids[nm] = g;
    if (f->adjoints[a][0]) env.grids[f->adjoints[a]] = b;
  }
  return env;
}

// The oracle on copies of env's grids; returns the grids by name.
static std::map<std::string, std::vector<double>> oracle(int fam, const sgb::Env& env,
                                                         bool adjoint, bool f32) {
  const sg_family* f = sg_family_get(fam);
  std::map<std::string, std::vector<double>> g;
  for (const auto& kv : env.grids) {
    g[kv.first] = kv.second.data();
    if (f32)
      for (double& v : g[kv.first]) v = (double)(float)v;
  }
  sg_env e{};
  e.n = env.sizes.at("n");
  for (int s = 0; s < f->nscalars; s++) e.scalars[s] = env.scalars.at(f->scalars[s]);
  for (int a = 0; a < f->narrays; a++) {
    e.grid[a] = g[f->arrays[a]].data();
    if (f->adjoints[a][0]) e.adj[a] = g[f->adjoints[a]].data();
  }
  const int rc = adjoint ? sg_run_program(fam, &e) : sg_run_primal(fam, &e);
  CHECK(rc == 0);
  return g;
}

static void test_family(const char* name, long long n) {
  const int fam = sg_family_by_name(name);
  const sg_family* f = sg_family_get(fam);
  const sgb::Env env = make_env(fam, n, 7 + (unsigned)n);
  const sgb::Env before = env;

  // run_program: every non-output adjoint at 1e-12 (fp64)
  const sgb::Env out = sgb::run_program(name, env);
  const auto want = oracle(fam, env, true, false);
  for (int a = 0; a < f->narrays; a++) {
    if (!f->adjoints[a][0] || a == f->output) continue;
    const double e = compare(out.grids.at(f->adjoints[a]), want.at(f->adjoints[a]));
    CHECK(e <= 1e-12);
    if (e > 1e-12) std::fprintf(stderr, "  %s n=%lld %s: %.3e\n", name, n, f->adjoints[a], e);
  }
  // the input Env is untouched (interp.hpp: const Env& in, copy out)
  for (const auto& kv : before.grids) CHECK(env.grids.at(kv.first).data() == kv.second.data());

  // run_scatter_adjoint agrees with the gather form at 1e-12 (verify_problem)
  const sgb::Env sc = sgb::run_scatter_adjoint(name, env);
  for (int a = 0; a < f->narrays; a++) {
    if (!f->adjoints[a][0] || a == f->output) continue;
    CHECK(compare(sc.grids.at(f->adjoints[a]), out.grids.at(f->adjoints[a]).data()) <= 1e-12);
  }

  // run_nest (primal) at 1e-12
  const sgb::Env pr = sgb::run_nest(name, env);
  const auto wp = oracle(fam, env, false, false);
  CHECK(compare(pr.grids.at(f->arrays[f->output]), wp.at(f->arrays[f->output])) <= 1e-12);

  // fp32 device precision against the oracle on the fp32-rounded inputs
  const sgb::Env o32 = sgb::run_program(name, env, sgb::Precision::f32);
  const auto w32 = oracle(fam, env, true, true);
  for (int a = 0; a < f->narrays; a++) {
    if (!f->adjoints[a][0] || a == f->output) continue;
    CHECK(compare(o32.grids.at(f->adjoints[a]), w32.at(f->adjoints[a])) <= 1e-5);
  }
}

template <typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const sgb::Error&) {
    return true;
  }
  return false;
}

// `makeenv <family> <n> <seed>`: the digest oracle/ref/ref_harness.cpp prints
// for the reference's make_env, here for sgb::make_env (host only, no GPU).
static int cmd_makeenv(const char* family, long long n, unsigned long long seed) {
  const sgb::Env env = sgb::make_env(family, {{"n", n}}, seed);
  char buf[64];
  auto num = [&](double v) {
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return std::string(buf);
  };
  std::string os = "{\"scalars\":{";
  bool first = true;
  for (const auto& kv : env.scalars) {
    os += std::string(first ? "" : ",") + "\"" + kv.first + "\":" + num(kv.second);
    first = false;
  }
  os += "},\"grids\":{";
  first = true;
  for (const auto& kv : env.grids) {
    const std::vector<double>& d = kv.second.data();
    double sum = 0, sq = 0;
    for (double x : d) sum += x, sq += x * x;
    os += std::string(first ? "" : ",") + "\"" + kv.first + "\":[" + std::to_string(d.size()) +
          "," + num(sum) + "," + num(sq) + "," + num(d.empty() ? 0 : d.front()) + "," +
          num(d.empty() ? 0 : d[d.size() / 2]) + "," + num(d.empty() ? 0 : d.back()) + "]";
    first = false;
  }
  std::printf("%s}}\n", os.c_str());
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 5 && std::string(argv[1]) == "makeenv")
    return cmd_makeenv(argv[2], std::atoll(argv[3]), std::strtoull(argv[4], nullptr, 10));
  if (argc >= 6 && std::string(argv[1]) == "verify") {  // verify <family> <n> <seed> <trials>
    const sgb::VerifyReport rep = sgb::verify_problem(
        argv[2], {{"n", std::atoll(argv[3])}}, std::strtoull(argv[4], nullptr, 10),
        std::atoi(argv[5]), true);
    std::fputs(rep.json_text().c_str(), stdout);
    std::fputs(rep.text().c_str(), stderr);
    return rep.pass() ? 0 : 1;
  }
  test_family("wave1d", 257);
  test_family("wave3d_c", 20);
  test_family("wave3d_c2", 17);
  test_family("burgers2d", 64);
  test_family("wave3d_r4", 36);
  test_family("wave3d_r4", 40);

  // errors: guard violation, missing grid, wrong shape, unsupported problem
  const sgb::Env small = make_env(SG_WAVE3D_R4, 12, 1);  // n - 9 < 8 (adjoint.cpp:134-143)
  CHECK(throws([&] { sgb::run_program("wave3d_r4", small); }));
  sgb::Env missing = make_env(SG_BURGERS2D, 16, 2);
  missing.grids.erase("u_b");
  CHECK(throws([&] { sgb::run_program("burgers2d", missing); }));
  sgb::Env shape = make_env(SG_BURGERS2D, 16, 3);
  shape.grids["u_1"] = sgb::DenseGrid({15, 16});
  CHECK(throws([&] { sgb::run_program("burgers2d", shape); }));
  CHECK(throws([&] { sgb::run_program("lap1d", small); }));
  CHECK(throws([&] { sgb::DenseGrid({4, 4}).flat({4, 0}); }));

  // program-keyed dispatch: the family's own program runs its kernels (same
  // result as the name-keyed call); an edited program is refused
  {
    const sgb::Env env = make_env(SG_WAVE3D_R4, 36, 11);
    const sgb::Program prog = sgb::Program::of("wave3d_r4");
    CHECK(prog.family() == "wave3d_r4");
    const sgb::Env a = sgb::run_program(prog, env), b = sgb::run_program("wave3d_r4", env);
    CHECK(a.grids.at("c_b").data() == b.grids.at("c_b").data());
    CHECK(a.grids.at("u_1_b").data() == b.grids.at("u_1_b").data());
    sgb::Program edited = prog;  // one partial's weight changed
    const auto at = edited.text.find("partial ");
    CHECK(at != std::string::npos);
    edited.text.insert(at + 8, "1.01*");
    CHECK(throws([&] { sgb::run_program(edited, env); }));
    sgb::Program bounds = prog;  // another primal box
    const auto g = bounds.text.find("guard n - 9");
    CHECK(g != std::string::npos);
    bounds.text.replace(g, 11, "guard n - 8");
    CHECK(throws([&] { (void)bounds.family(); }));
    CHECK(throws([&] { (void)sgb::Program::of("lap1d"); }));
  }

  // compare_grids: the reference's metric, NaN terms ignored, shapes checked
  {
    sgb::DenseGrid a({3, 4}), b({3, 4});
    for (std::size_t i = 0; i < 12; i++) a.data()[i] = b.data()[i] = 0.5 * (double)i - 2.0;
    a.data()[5] += 3e-3;  // b[5] = 0.5: err = 3e-3 / 1.5
    const sgb::GridCompare c = sgb::compare_grids(a, b, 1e-2);
    CHECK(std::fabs(c.max_rel_err - 3e-3 / 1.5) < 1e-15 && c.pass);
    CHECK(!sgb::compare_grids(a, b, 1e-3).pass);
    a.data()[7] = std::nan("");
    CHECK(std::fabs(sgb::compare_grids(a, b, 1e-2).max_rel_err - 3e-3 / 1.5) < 1e-15);
    CHECK(throws([&] { sgb::compare_grids(a, sgb::DenseGrid({4, 3}), 1.0); }));
  }
  // dot_product_test on a caller's Env, and its argument check
  {
    const sgb::Env env = sgb::make_env("wave3d_c2", {{"n", 14}}, 5);
    const sgb::DotReport d = sgb::dot_product_test("wave3d_c2", env, 2);
    CHECK(d.pass && d.trials == 2 && d.threshold == 1e-4 && d.max_rel_err < 1e-6);
    CHECK(throws([&] { sgb::dot_product_test("wave3d_c2", env, 0); }));
  }

  std::printf("host_api: %d checks, %d failures\n", g_checks, g_failures);
  return g_failures ? 1 : 0;
}
