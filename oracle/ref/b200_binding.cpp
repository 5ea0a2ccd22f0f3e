// b200_binding.cpp — the reference-side binding INTEGRATION.md describes,
// compiled against the UNMODIFIED reference headers (proj/include) and used by
// ref_harness' `b200` / `canon` commands to check the B200 library through the
// reference's own in-memory API types (AdjointProgram, Env, DenseGrid;
// adjoint.hpp:37-45, interp.hpp:14-59).
//
// run_program_b200(program, env) has the contract of the reference's
// run_program(program, env) (interp.hpp:59): it returns a modified copy of env
// with every adjoint array accumulated.  Dispatch is keyed on the PROGRAM, not
// on a name: the program's canonical text (b200_program_text, below) is
// handed to sgb_program_family(), which answers with the family whose
// hand-tuned kernels compute exactly that program (same counters, terms,
// offsets, partials, seeds, valid boxes, nests, guards) or NULL -- then this
// binding throws stencilgrad::Error, so no program is ever silently given a
// hard-coded stencil (the general path for other programs is the NVRTC
// emitter, paper_1907_02818_b200/emitter.py).  The B200 library is loaded
// with dlopen so the harness builds without a GPU; SGB_LIB names it (default:
// the in-tree .so).
#include <dlfcn.h>

#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "stencilgrad/adjoint.hpp"
#include "stencilgrad/interp.hpp"

namespace stencilgrad {

namespace {

struct B200 {
  void* h = nullptr;
  void* (*plan_create)(const char*, int, int) = nullptr;
  void (*plan_destroy)(void*) = nullptr;
  int (*plan_run)(void*, const double*, void**, void*) = nullptr;
  const char* (*last_error)() = nullptr;
  const char* (*program_family)(const char*) = nullptr;
  const char* (*family_signature)(const char*) = nullptr;
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
    b.program_family =
        reinterpret_cast<const char* (*)(const char*)>(dlsym(b.h, "sgb_program_family"));
    b.family_signature =
        reinterpret_cast<const char* (*)(const char*)>(dlsym(b.h, "sgb_family_signature"));
    if (!b.plan_create || !b.plan_run || !b.plan_destroy || !b.last_error ||
        !b.program_family || !b.family_signature)
      throw Error("B200 library lacks the sgb_plan_* / sgb_program_* entry points");
  }
  return b;
}

std::string join_ranges(const std::vector<Range>& rs) {
  std::string s;
  for (std::size_t i = 0; i < rs.size(); i++)
    s += (i ? "," : "") + rs[i].lo.str() + ":" + rs[i].hi.str();
  return s;
}

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char ch : s) {
    if (ch == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur += ch;
    }
  }
  if (!cur.empty()) out.push_back(cur);
  return out;
}

}  // namespace

// Canonical text of an AdjointProgram (format documented in
// include/stencilgrad_b200.h at sgb_program_family): everything run_program
// executes -- counters, extent guards, every term (active read, offset,
// adjoint array, seed array and its lhs permutation, partial printed by
// to_input_string, expr.hpp:92), every shifted statement's valid box, every
// nest (bounds, term list, core flag) and the core index.
std::string b200_program_text(const AdjointProgram& prog) {
  std::ostringstream os;
  os << "sgb-program 1\ncounters";
  for (const auto& c : prog.counters) os << " " << c;
  os << "\n";
  for (const auto& g : prog.extent_guards) os << "guard " << g.first.str() << " >= " << g.second << "\n";
  for (std::size_t t = 0; t < prog.terms.size(); t++) {
    const AdjointTerm& at = prog.terms[t];
    os << "term " << t << " read " << at.input.array << " offset";
    for (long long o : at.input.offset) os << " " << o;
    os << " adjoint " << at.adjoint_array << " seed " << at.seed_array;
    for (const auto& c : at.seed_lhs) os << "[" << c << "]";
    os << " partial " << to_input_string(at.partial) << "\n";
  }
  for (std::size_t t = 0; t < prog.shifted.size(); t++)
    os << "valid " << t << " " << join_ranges(prog.shifted[t].valid) << "\n";
  for (const auto& nest : prog.nests) {
    os << "nest " << join_ranges(nest.nest.bounds) << " terms";
    for (std::size_t t : nest.terms) os << " " << t;
    os << (nest.core ? " core" : "") << "\n";
  }
  os << "core " << prog.core_index << "\n";
  return os.str();
}

// The family whose hand-tuned B200 kernels compute `prog`, or "" (reason in
// *why).
std::string b200_program_family(const AdjointProgram& prog, std::string* why) {
  const B200& b = lib();
  const std::string text = b200_program_text(prog);
  const char* fam = b.program_family(text.c_str());
  if (!fam) {
    if (why) *why = b.last_error();
    return "";
  }
  return fam;
}

Env run_program_b200(const AdjointProgram& prog, const Env& env) {
  std::string why;
  const std::string family = b200_program_family(prog, &why);
  if (family.empty())
    throw Error("no B200 kernel computes this AdjointProgram (" + why +
                "); lower it with the NVRTC emitter instead");
  const B200& b = lib();
  // the family's generated prototype: "sizes;scalars;arrays" in the order of
  // the reference emitter's signature (codegen.cpp:198-230)
  const auto sig = split(b.family_signature(family.c_str()), ';');
  if (sig.size() != 3) throw Error("bad signature for " + family);
  Env out = env;
  const long long n = env.sizes.at(split(sig[0], ',').at(0));
  void* plan = b.plan_create(family.c_str(), static_cast<int>(n), 8);  // fp64 kernels
  if (!plan) throw Error(std::string("sgb_plan_create: ") + b.last_error());
  std::vector<double> scalars;
  for (const auto& s : split(sig[1], ',')) scalars.push_back(env.scalars.at(s));
  std::vector<void*> arrays;
  for (const auto& a : split(sig[2], ',')) arrays.push_back(out.grids.at(a).data().data());
  const int rc = b.plan_run(plan, scalars.data(), arrays.data(), nullptr);
  const std::string err = rc ? b.last_error() : "";
  b.plan_destroy(plan);
  if (rc == 1) throw Error("minimum extent violated");
  if (rc != 0) throw Error("B200 gather adjoint failed: " + err);
  return out;
}

}  // namespace stencilgrad
