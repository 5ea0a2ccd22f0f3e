// b200_binding.cpp — the reference-side binding INTEGRATION.md describes,
// compiled against the UNMODIFIED reference headers (proj/include) and used by
// ref_harness' `b200` command to check the B200 library through the
// reference's own in-memory API types (Problem, Env, DenseGrid; interp.hpp).
//
// run_program_b200(p, env) has the contract of
// run_program(assemble_adjoint(p), env) (interp.hpp:59): it returns a modified
// copy of env with every adjoint array accumulated; unsupported problems throw
// stencilgrad::Error.  The B200 library is loaded with dlopen so the harness
// builds without a GPU; SGB_LIB names it (default: the in-tree .so).
#include <dlfcn.h>

#include <cstdlib>
#include <string>
#include <vector>

#include "stencilgrad/interp.hpp"

namespace stencilgrad {

namespace {

struct B200 {
  void* h = nullptr;
  void* (*plan_create)(const char*, int, int) = nullptr;
  void (*plan_destroy)(void*) = nullptr;
  int (*plan_run)(void*, const double*, void**, void*) = nullptr;
  const char* (*last_error)() = nullptr;
};

const B200& lib() {
  static B200 b;
  if (!b.h) {
    const char* path = std::getenv("SGB_LIB");
    b.h = dlopen(path ? path : "libstencilgrad_b200.so", RTLD_NOW | RTLD_LOCAL);
    if (!b.h) throw Error(std::string("cannot load the B200 library: ") + dlerror());
    b.plan_create = reinterpret_cast<void* (*)(const char*, int, int)>(dlsym(b.h, "sgb_plan_create"));
    b.plan_destroy = reinterpret_cast<void (*)(void*)>(dlsym(b.h, "sgb_plan_destroy"));
    b.plan_run = reinterpret_cast<int (*)(void*, const double*, void**, void*)>(
        dlsym(b.h, "sgb_plan_run_adjoint_host"));
    b.last_error = reinterpret_cast<const char* (*)()>(dlsym(b.h, "sgb_last_error"));
    if (!b.plan_create || !b.plan_run || !b.plan_destroy || !b.last_error)
      throw Error("B200 library lacks the sgb_plan_* entry points");
  }
  return b;
}

// the generated prototype's array order: declaration order, each primal array
// followed by its adjoint, only arrays the adjoint references (codegen.cpp:198-211)
std::vector<std::string> prototype_arrays(const std::string& family) {
  if (family == "wave1d") return {"c", "c_b", "u", "u_b", "u_prev_b", "u_next_b"};
  if (family == "wave3d_c" || family == "wave3d_c2")
    return {"c", "c_b", "u_1", "u_1_b", "u_2_b", "u_b"};
  if (family == "burgers2d") return {"u_1", "u_1_b", "u_b"};
  if (family == "wave3d_r4") return {"c", "c_b", "u_1", "u_1_b", "u_b"};
  throw Error("no B200 kernel for problem '" + family + "'");
}

}  // namespace

Env run_program_b200(const Problem& p, const Env& env) {
  const auto names = prototype_arrays(p.name);
  const B200& b = lib();
  Env out = env;
  const long long n = env.sizes.at("n");
  void* plan = b.plan_create(p.name.c_str(), static_cast<int>(n), 8);  // fp64 kernels
  if (!plan) throw Error(std::string("sgb_plan_create: ") + b.last_error());
  std::vector<double> scalars;
  for (const auto& s : p.scalars) scalars.push_back(env.scalars.at(s));
  std::vector<void*> arrays;
  for (const auto& a : names) arrays.push_back(out.grids.at(a).data().data());
  const int rc = b.plan_run(plan, scalars.data(), arrays.data(), nullptr);
  const std::string err = rc ? b.last_error() : "";
  b.plan_destroy(plan);
  if (rc == 1) throw Error("minimum extent violated");
  if (rc != 0) throw Error("B200 gather adjoint failed: " + err);
  return out;
}

}  // namespace stencilgrad
