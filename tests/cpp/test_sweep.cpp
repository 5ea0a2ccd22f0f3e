// The host-state sweeps of INTEGRATION.md section 1 from plain C++ over the C
// ABI (include/stencilgrad_b200.h): sgb_plan_sweep_begin / _step_host / _end
// against what a caller of the per-step reference ABI gets
// (sgb_plan_run_adjoint_host per step + its own zeroing / rotation), bit for
// bit.  Needs a GPU; built and run by tests/test_sweep_cpp.py.
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "stencilgrad_b200.h"

static int g_checks = 0, g_failures = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    g_checks++;                                                                  \
    if (!(cond)) {                                                               \
      g_failures++;                                                              \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #cond); \
    }                                                                            \
  } while (0)

using Grid = std::vector<float>;

static Grid draw(size_t count, std::mt19937_64& rng, float lo, float hi, bool normal) {
  Grid g(count);
  std::normal_distribution<float> N(0.f, 1.f);
  std::uniform_real_distribution<float> U(lo, hi);
  for (float& v : g) v = normal ? N(rng) : U(rng);
  return g;
}

static bool same(const Grid& a, const Grid& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(float)) == 0;
}

// cfg 5's protocol: independent steps, u_1_b = the step's adjoint, c_b accumulated
static void independent_steps(int n, int T) {
  const size_t count = (size_t)n * n * n;
  std::mt19937_64 rng(1234 + n);
  const Grid c = draw(count, rng, 1.5f, 4.5f, false), c_b0 = draw(count, rng, 0, 0, true);
  std::vector<Grid> u_1, u_b;
  for (int t = 0; t < T; t++) {
    u_1.push_back(draw(count, rng, 0, 0, true));
    u_b.push_back(draw(count, rng, 0, 0, true));
  }
  const double D = 0.01;
  sgb_plan* plan = sgb_plan_create("wave3d_r4", n, 4);
  CHECK(plan != nullptr);
  // the caller of the per-step ABI: memset(u_1_b); wave3d_r4_b(...) on host arrays
  Grid ref_cb = c_b0;
  std::vector<Grid> ref_u1b;
  for (int t = 0; t < T; t++) {
    Grid cc = c, x = u_1[t], s = u_b[t], out(count, 0.f);
    void* a[5] = {cc.data(), ref_cb.data(), x.data(), out.data(), s.data()};
    CHECK(sgb_plan_run_adjoint_host(plan, &D, a, nullptr) == 0);
    ref_u1b.push_back(out);
  }
  // the sweep
  Grid cc = c, cb = c_b0, out(count);
  void* a[5] = {cc.data(), cb.data(), nullptr, nullptr, nullptr};
  CHECK(sgb_plan_sweep_step_host(plan, &D, a, nullptr) != 0);  // no sweep begun
  CHECK(sgb_plan_sweep_begin(plan, a, nullptr) == 0);
  {  // the per-step entry would overwrite the resident arrays: refused while a sweep is open
    Grid x = u_1[0], s = u_b[0];
    void* b[5] = {cc.data(), cb.data(), x.data(), out.data(), s.data()};
    CHECK(sgb_plan_run_adjoint_host(plan, &D, b, nullptr) != 0);
  }
  for (int t = 0; t < T; t++) {
    a[2] = u_1[t].data();
    a[3] = out.data();
    a[4] = u_b[t].data();
    CHECK(sgb_plan_sweep_step_host(plan, &D, a, nullptr) == 0);
    CHECK(same(out, ref_u1b[t]));
  }
  CHECK(sgb_plan_sweep_end(plan, a, nullptr) == 0);
  CHECK(same(cb, ref_cb));
  CHECK(sgb_plan_sweep_end(plan, a, nullptr) != 0);  // already ended
  sgb_plan_destroy(plan);
}

// cfg 2's protocol: carried steps, the adjoints rotate
static void carried_steps(int n, int T) {
  const size_t count = (size_t)n * n * n;
  std::mt19937_64 rng(99 + n);
  const Grid c = draw(count, rng, 1.5f, 4.5f, false);
  Grid cb = draw(count, rng, 0, 0, true), u1b = draw(count, rng, 0, 0, true),
       u2b = draw(count, rng, 0, 0, true), ub = draw(count, rng, 0, 0, true);
  std::vector<Grid> u_1;
  for (int t = 0; t < T; t++) u_1.push_back(draw(count, rng, 0, 0, true));
  const double D = 0.1;
  sgb_plan* plan = sgb_plan_create("wave3d_c", n, 4);
  CHECK(plan != nullptr);
  Grid r_cb = cb, r_u1b = u1b, r_u2b = u2b, r_ub = ub;
  for (int t = 0; t < T; t++) {
    Grid cc = c, x = u_1[t];
    void* a[6] = {cc.data(), r_cb.data(), x.data(), r_u1b.data(), r_u2b.data(), r_ub.data()};
    CHECK(sgb_plan_run_adjoint_host(plan, &D, a, nullptr) == 0);
    r_ub.swap(r_u1b);   // seed <- u_1_b
    r_u1b.swap(r_u2b);  // u_1_b <- u_2_b
    std::fill(r_u2b.begin(), r_u2b.end(), 0.f);
  }
  Grid cc = c;
  void* a[6] = {cc.data(), cb.data(), nullptr, u1b.data(), u2b.data(), ub.data()};
  CHECK(sgb_plan_sweep_begin(plan, a, nullptr) == 0);
  for (int t = 0; t < T; t++) {
    a[2] = u_1[t].data();
    CHECK(sgb_plan_sweep_step_host(plan, &D, a, nullptr) == 0);
  }
  CHECK(sgb_plan_sweep_end(plan, a, nullptr) == 0);
  CHECK(same(cb, r_cb) && same(u1b, r_u1b) && same(u2b, r_u2b) && same(ub, r_ub));
  sgb_plan_destroy(plan);
}

int main() {
  independent_steps(136, 3);
  independent_steps(40, 2);
  carried_steps(132, 4);
  // families without a sweep form are refused
  sgb_plan* b = sgb_plan_create("burgers2d", 64, 8);
  void* none[3] = {nullptr, nullptr, nullptr};
  CHECK(b && sgb_plan_sweep_begin(b, none, nullptr) != 0);
  sgb_plan_destroy(b);
  std::printf("sweep: %d checks, %d failures\n", g_checks, g_failures);
  return g_failures ? 1 : 0;
}
