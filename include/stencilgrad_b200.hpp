// stencilgrad_b200.hpp — C++ host API above the C ABI (stencilgrad_b200.h).
//
// Mirrors the reference's in-memory API (proj/include/stencilgrad/interp.hpp):
//   Env run_nest(const StencilLoopNest&, const Env&)           interp.hpp:56
//   Env run_program(const AdjointProgram&, const Env&)         interp.hpp:59
//   Env run_scatter_adjoint(const Problem&, const Env&)        interp.hpp:63
//   Env make_env(const Problem&, sizes, seed)                  interp.hpp:45
//   GridCompare compare_grids(a, b, rel_tol)                   interp.hpp:71
//   DotReport dot_product_test(p, program, env, trials)        interp.hpp:83
//   VerifyReport verify_problem(p, sizes, seed, trials, fd)    interp.hpp:102
// with the same argument meaning and error behaviour: the input Env is taken
// by const& and left untouched, an updated copy is returned; adjoint grids
// are accumulated (+=); a minimum-extent guard violation, a missing grid or a
// grid of the wrong shape throws sgb::Error (the reference's
// stencilgrad::Error).  The problem is named by family (wave1d, wave3d_c,
// wave3d_c2, burgers2d, wave3d_r4): for these the reference's Problem /
// AdjointProgram is fixed by the spec (oracle/specs/<family>.json), and the
// B200 kernels are its compiled form.  Grids are host fp64 like the
// reference's DenseGrid; Precision::f32 computes in fp32 on the device (the
// BASELINE precision of the 3D configs) and converts back.  Every call runs on
// the GPU (upload, the <name>[_b|_scatter_b] kernel, download); there is no
// CPU path.
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace sgb {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Row-major multidimensional array of doubles (stencilgrad::DenseGrid,
// interp.hpp:14-33).
class DenseGrid {
 public:
  DenseGrid() = default;
  explicit DenseGrid(std::vector<long long> shape);

  const std::vector<long long>& shape() const { return shape_; }
  std::vector<double>& data() { return data_; }
  const std::vector<double>& data() const { return data_; }

  bool in_bounds(const std::vector<long long>& idx) const;
  std::size_t flat(const std::vector<long long>& idx) const;
  double at(const std::vector<long long>& idx) const { return data_[flat(idx)]; }
  double& at(const std::vector<long long>& idx) { return data_[flat(idx)]; }

 private:
  std::vector<long long> shape_;
  std::vector<double> data_;
};

// stencilgrad::Env (interp.hpp:35-40): sizes ("n"), scalars by name, grids by
// array / adjoint name.
struct Env {
  std::map<std::string, long long> sizes;
  std::map<std::string, double> scalars;
  std::map<std::string, DenseGrid> grids;
  std::uint64_t seed = 0;  // make_env's seed (dot_product_test derives its draws from it)
};

enum class Precision { f64, f32 };

// An AdjointProgram (adjoint.hpp:37-45) in the canonical text form of
// sgb_program_family (stencilgrad_b200.h): what run_program executes.
// Program::of(family) is the program the family's kernels compute (the
// reference front end's assemble_adjoint of oracle/specs/<family>.json).
struct Program {
  std::string text;
  static Program of(const std::string& family);
  // the family whose hand-tuned kernels compute exactly this program; throws
  // Error (naming the first differing line) when there is none
  std::string family() const;
};

// Gather adjoint of `program` (run_program(const AdjointProgram&, const Env&),
// interp.hpp:59): dispatched on the program itself -- a program no hand-tuned
// family computes throws Error instead of running a hard-coded stencil.
Env run_program(const Program& program, const Env& env, Precision p = Precision::f64);

// Primal (run_nest semantics): the output grid updated on the primal box.
Env run_nest(const std::string& family, const Env& env, Precision p = Precision::f64);
// Gather adjoint (run_program semantics): guards first, then every input
// adjoint accumulated over the core + boundary regions.
Env run_program(const std::string& family, const Env& env, Precision p = Precision::f64);
// Atomic-scatter adjoint (run_scatter_adjoint semantics, ablation).
Env run_scatter_adjoint(const std::string& family, const Env& env,
                        Precision p = Precision::f64);

// make_env (interp.hpp:42-45, interp.cpp:266-288): the reference's reproducible
// environment for `family`, value for value -- one mt19937_64 seeded with
// `seed` feeds a normal(0,1) stream: the scalars in spec order, the primal
// grids in declaration order, then the output's adjoint seed; input adjoints
// start at zero (inactive arrays get no adjoint).  Host-side input
// generation; pinned to the reference's own make_env by tests/golden/
// ref_make_env.json.
Env make_env(const std::string& family, const std::map<std::string, long long>& sizes,
             std::uint64_t seed);

// compare_grids (interp.hpp:66-71): max over elements of |a - b| / (1 + |b|)
// (NaN terms never raise the maximum, as with the reference's std::max), pass
// iff <= rel_tol; a shape mismatch throws.  Reduced on the device
// (sgb_compare_f64).
struct GridCompare {
  double max_rel_err = 0.0;
  bool pass = false;
};
GridCompare compare_grids(const DenseGrid& a, const DenseGrid& b, double rel_tol);

// dot_product_test (interp.hpp:73-84, interp.cpp:300-389): <J v, w> = <v, J^T w>
// with Gaussian probes, a central finite difference of the PRIMAL KERNEL on the
// left and the GATHER ADJOINT KERNEL on the right (fp64 on the device); the
// same draws as the reference (mix_seed(env.seed, trial, attempt)), the same
// step h = 1e-5 (1 + max |input|), the same redraw when a min/max argument is
// within 1e-3 of a tie (burgers2d), threshold 1e-4 (every family is nonlinear
// in its active inputs).
struct DotReport {
  double max_rel_err = 0.0;
  double threshold = 0.0;
  int trials = 0;
  bool pass = false;
};
DotReport dot_product_test(const std::string& family, const Env& env, int trials);

// verify_problem (interp.hpp:86-103, interp.cpp:413-435): "oracle-equivalence"
// = the gather adjoint kernel against the atomic-scatter adjoint kernel on
// make_env(family, sizes, seed) at 1e-12, plus (fd) "dot-product".  text() and
// json_text() print the reference's report layout.
struct CheckLine {
  std::string name;
  double metric = 0.0;
  double threshold = 0.0;
  bool pass = false;
};
struct VerifyReport {
  std::vector<CheckLine> checks;
  bool pass() const;
  std::string text() const;
  std::string json_text() const;
};
VerifyReport verify_problem(const std::string& family,
                            const std::map<std::string, long long>& sizes, std::uint64_t seed,
                            int trials, bool fd);

// Array names a call reads / writes, in the C ABI (reference emitter) order.
std::vector<std::string> array_params(const std::string& family, const std::string& kind);

}  // namespace sgb
