// stencilgrad_b200.hpp — C++ host API above the C ABI (stencilgrad_b200.h).
//
// Mirrors the reference's in-memory API (proj/include/stencilgrad/interp.hpp):
//   Env run_nest(const StencilLoopNest&, const Env&)           interp.hpp:56
//   Env run_program(const AdjointProgram&, const Env&)         interp.hpp:59
//   Env run_scatter_adjoint(const Problem&, const Env&)        interp.hpp:63
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

// Array names a call reads / writes, in the C ABI (reference emitter) order.
std::vector<std::string> array_params(const std::string& family, const std::string& kind);

}  // namespace sgb
