// ref_harness — TEST INFRASTRUCTURE ONLY (never on the product path).
//
// Drives the UNMODIFIED reference library (`stencilgrad`, compiled from the
// sources under /root/reference/proj/src by oracle/ref/Makefile into
// oracle/_ref/) so that the repo's own oracle restatement (oracle/sg_oracle.c)
// and the CUDA path can be pinned against the reference's own semantics:
//
//   info   <spec> <n>                         program structure as JSON
//                                             (assemble_adjoint, adjoint.cpp:152-163)
//   run    <spec> <n> <in_dir> <out_dir> S=v  run_nest / run_program /
//                                             run_scatter_adjoint (interp.cpp:183-228)
//                                             on raw fp64 grids read from in_dir
//   verify <spec> <n> <seed> <trials>         verify_problem (interp.cpp:413-435)
//   makeenv <spec> <n> <seed>                 make_env (interp.cpp:266-288): scalars
//                                             and per-grid digests as JSON
//   b200   <spec> <n> <in_dir> S=v            run_program vs run_program_b200 (the
//                                             INTEGRATION.md binding, b200_binding.cpp)
//                                             on the same Env; prints the max
//                                             compare_grids error as JSON, or
//                                             {"error": ...} (exit 3) when the
//                                             binding refuses the program
//   canon  <spec>                             the program's canonical text
//                                             (b200_program_text), exported as
//                                             paper_1907_02818_b200/programs/<name>.canon
//   timeloop <spec> <n> <T> <in_dir> <out_dir> S=v
//                                             the adjoint of a whole time loop
//                                             u^{t+1} = F(u^t, u^{t-1}), J = <w, u^T>,
//                                             composed from the reference's own
//                                             run_nest (forward) and run_program
//                                             (reverse, interp.cpp:183-198); <spec>
//                                             must have u_2 active (adjoint u_2_b);
//                                             reads c, u0, u1, w; writes u0_b, u1_b,
//                                             c_b (the pin of drivers.time_loop_adjoint)
//   match  <spec>                             the family the B200 library's
//                                             sgb_program_family() assigns to the
//                                             program (no GPU needed), JSON
//   spec   <spec>                             serialize_spec (specfile.cpp:208-240)
//   emit   <spec> <out_dir>                   emit_primal / emit_adjoint /
//                                             emit_scatter_adjoint with restrict,
//                                             exactly as cmd_bench does
//                                             (tools/stencilgrad.cpp:285-301)
//
// <spec> is a path to a JSON spec, "example:<name>" for a bundled example
// (examples.cpp:79), or "opaque:<name>" for an opaque-call problem built
// through the reference's expression builders (the JSON front end has no
// syntax for opaque calls, parser.cpp:210): "opaque:paper2d" is the paper's
// f(a = u[i-1][j], b = u[i][j-1]) example, "opaque:line1d" a 1D
// two-argument call; `emit` declares C prototypes for f / f_d_a / f_d_b (g /
// g_d_x / g_d_y) as the reference requires (codegen.cpp:153-158, :290-300).  Grids are raw little-endian fp64, row-major, named
// <array>.f64.  Nothing here is shipped or timed.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "stencilgrad/adjoint.hpp"
#include "stencilgrad/codegen.hpp"
#include "stencilgrad/examples.hpp"
#include "stencilgrad/interp.hpp"
#include "stencilgrad/parser.hpp"
#include "stencilgrad/specfile.hpp"

namespace sg = stencilgrad;

namespace stencilgrad {  // b200_binding.cpp
Env run_program_b200(const AdjointProgram& prog, const Env& env);
std::string b200_program_text(const AdjointProgram& prog);
std::string b200_program_family(const AdjointProgram& prog, std::string* why);
}

static std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw sg::Error("cannot read " + path);
  std::ostringstream os;
  os << in.rdbuf();
  return os.str();
}

static sg::ExprPtr P(const char* text) {
  std::string err;
  auto e = sg::parse_expr(text, &err);
  if (!e) throw sg::Error(std::string("parse_expr: ") + err);
  return e;
}

static sg::Problem opaque_problem(const std::string& name) {
  std::string spec;
  sg::ExprPtr rhs;
  if (name == "paper2d") {
    spec = R"({"name": "opq2d", "counters": ["i", "j"],
      "bounds": {"i": ["1", "n - 2"], "j": ["1", "n - 2"]}, "sizes": ["n"], "scalars": ["a"],
      "arrays": {"u": {"rank": 2, "shape": ["n", "n"], "active": true, "adjoint": "u_b",
                       "role": "input"},
                 "c": {"rank": 2, "shape": ["n", "n"], "active": false, "role": "coefficient"},
                 "r": {"rank": 2, "shape": ["n", "n"], "active": true, "adjoint": "r_b",
                       "role": "output"}},
      "lhs": "r[i][j]", "mode": "=", "rhs": "a*u[i][j]"})";
    // r = c * f(a = u[i-1][j], b = u[i][j-1]) + a * u
    rhs = sg::add({sg::mul({P("c[i][j]"),
                            sg::opaque_call("f", {{"a", P("u[i - 1][j]")}, {"b", P("u[i][j - 1]")}})}),
                   P("a*u[i][j]")});
  } else if (name == "line1d") {
    spec = R"({"name": "opq1d", "counters": ["i"], "bounds": {"i": ["2", "n - 3"]},
      "sizes": ["n"], "scalars": ["a"],
      "arrays": {"u": {"rank": 1, "shape": ["n"], "active": true, "adjoint": "u_b",
                       "role": "input"},
                 "r": {"rank": 1, "shape": ["n"], "active": true, "adjoint": "r_b",
                       "role": "output"}},
      "lhs": "r[i]", "mode": "+=", "rhs": "a*u[i]"})";
    // r += g(x = u[i-2], y = u[i+1]) * u[i] + a * g(x = u[i], y = u[i])
    rhs = sg::add({sg::mul({sg::opaque_call("g", {{"x", P("u[i - 2]")}, {"y", P("u[i + 1]")}}),
                            P("u[i]")}),
                   sg::mul({P("a"), sg::opaque_call("g", {{"x", P("u[i]")}, {"y", P("u[i]")}})})});
  } else {
    throw sg::Error("unknown opaque example " + name);
  }
  auto r = sg::parse_spec(spec);
  if (!r.problem) throw sg::Error("spec rejected:\n" + r.report.str());
  sg::Problem p = *r.problem;
  p.nest.body[0].rhs = rhs;
  return p;
}

static sg::Problem load(const std::string& spec) {
  if (spec.rfind("example:", 0) == 0) return sg::example_problem(spec.substr(8));
  if (spec.rfind("opaque:", 0) == 0) return opaque_problem(spec.substr(7));
  auto r = sg::parse_spec(slurp(spec));
  if (!r.problem) throw sg::Error("spec rejected:\n" + r.report.str());
  return *r.problem;
}

static std::vector<long long> shape_of(const sg::ArrayDecl& a,
                                       const std::map<std::string, long long>& sizes) {
  std::vector<long long> s;
  for (const auto& e : a.shape) s.push_back(e.eval(sizes));
  return s;
}

static void read_grid(const std::string& path, sg::DenseGrid& g) {
  std::ifstream in(path, std::ios::binary);
  if (!in) return;  // absent file: keep zeros
  in.read(reinterpret_cast<char*>(g.data().data()),
          static_cast<std::streamsize>(g.data().size() * sizeof(double)));
  if (!in) throw sg::Error("short read " + path);
}

static void write_grid(const std::string& path, const sg::DenseGrid& g) {
  std::ofstream out(path, std::ios::binary);
  out.write(reinterpret_cast<const char*>(g.data().data()),
            static_cast<std::streamsize>(g.data().size() * sizeof(double)));
}

static void print_range(std::ostream& os, const sg::Range& r, const std::map<std::string, long long>& sz) {
  os << "[" << r.lo.eval(sz) << "," << r.hi.eval(sz) << "]";
}

static int cmd_info(const sg::Problem& p, long long n) {
  std::map<std::string, long long> sz{{"n", n}};
  auto prog = sg::assemble_adjoint(p);
  std::ostringstream os;
  os << "{\"name\":\"" << p.name << "\",\"terms\":[";
  for (std::size_t t = 0; t < prog.terms.size(); t++) {
    if (t) os << ",";
    os << "{\"array\":\"" << prog.terms[t].input.array << "\",\"adjoint\":\""
       << prog.terms[t].adjoint_array << "\",\"offset\":[";
    for (std::size_t i = 0; i < prog.terms[t].input.offset.size(); i++)
      os << (i ? "," : "") << prog.terms[t].input.offset[i];
    os << "],\"partial\":\"" << sg::to_input_string(prog.terms[t].partial) << "\"}";
  }
  os << "],\"core_index\":" << prog.core_index << ",\"guards\":[";
  for (std::size_t g = 0; g < prog.extent_guards.size(); g++)
    os << (g ? "," : "") << "[" << prog.extent_guards[g].first.eval(sz) << ","
       << prog.extent_guards[g].second << "]";
  os << "],\"core_bounds\":[";
  auto cb = sg::core_bounds(prog.terms, p.nest);
  for (std::size_t i = 0; i < cb.size(); i++) {
    if (i) os << ",";
    print_range(os, cb[i], sz);
  }
  os << "],\"nests\":[";
  for (std::size_t k = 0; k < prog.nests.size(); k++) {
    if (k) os << ",";
    os << "{\"bounds\":[";
    for (std::size_t i = 0; i < prog.nests[k].nest.bounds.size(); i++) {
      if (i) os << ",";
      print_range(os, prog.nests[k].nest.bounds[i], sz);
    }
    os << "],\"terms\":[";
    for (std::size_t i = 0; i < prog.nests[k].terms.size(); i++)
      os << (i ? "," : "") << prog.nests[k].terms[i];
    os << "],\"core\":" << (prog.nests[k].core ? "true" : "false") << "}";
  }
  os << "]}\n";
  std::cout << os.str();
  return 0;
}

static sg::Env load_env(const sg::Problem& p, long long n, const std::string& in_dir, int argc,
                        char** argv) {
  sg::Env env;
  env.sizes["n"] = n;
  for (const auto& s : p.scalars) env.scalars[s] = 0.0;
  for (int a = 0; a < argc; a++) {
    std::string kv = argv[a];
    auto eq = kv.find('=');
    env.scalars[kv.substr(0, eq)] = std::strtod(kv.c_str() + eq + 1, nullptr);
  }
  for (const auto& a : p.arrays) {
    sg::DenseGrid g(shape_of(a, env.sizes));
    read_grid(in_dir + "/" + a.name + ".f64", g);
    env.grids[a.name] = g;
    if (a.active) {
      sg::DenseGrid gb(shape_of(a, env.sizes));
      read_grid(in_dir + "/" + a.adjoint + ".f64", gb);
      env.grids[a.adjoint] = gb;
    }
  }
  return env;
}

static int cmd_b200(const sg::Problem& p, long long n, const std::string& in_dir, int argc,
                    char** argv) {
  sg::Env env = load_env(p, n, in_dir, argc, argv);
  const auto prog = sg::assemble_adjoint(p);
  sg::Env ref = sg::run_program(prog, env);
  sg::Env gpu;
  try {
    gpu = sg::run_program_b200(prog, env);
  } catch (const sg::Error& e) {
    std::string msg = e.what();
    for (auto& ch : msg)
      if (ch == '"' || ch == '\\' || ch == '\n') ch = ' ';
    std::cout << "{\"name\":\"" << p.name << "\",\"error\":\"" << msg << "\"}\n";
    return 3;
  }
  const sg::ArrayDecl& out = sg::output_array(p);
  double worst = 0.0;
  std::ostringstream os;
  os << "{\"name\":\"" << p.name << "\",\"n\":" << n << ",\"arrays\":{";
  bool first = true;
  for (const auto& a : p.arrays) {
    if (!a.active || a.name == out.name) continue;
    auto c = sg::compare_grids(gpu.grids.at(a.adjoint), ref.grids.at(a.adjoint), 1e-12);
    worst = std::max(worst, c.max_rel_err);
    os << (first ? "" : ",") << "\"" << a.adjoint << "\":" << c.max_rel_err;
    first = false;
  }
  os << "},\"max_rel_err\":" << worst << "}\n";
  std::cout << os.str();
  return worst <= 1e-12 ? 0 : 1;
}

static int cmd_run(const sg::Problem& p, long long n, const std::string& in_dir,
                   const std::string& out_dir, int argc, char** argv) {
  sg::Env env;
  env.sizes["n"] = n;
  for (const auto& s : p.scalars) env.scalars[s] = 0.0;
  for (int a = 0; a < argc; a++) {
    std::string kv = argv[a];
    auto eq = kv.find('=');
    env.scalars[kv.substr(0, eq)] = std::strtod(kv.c_str() + eq + 1, nullptr);
  }
  for (const auto& a : p.arrays) {
    sg::DenseGrid g(shape_of(a, env.sizes));
    read_grid(in_dir + "/" + a.name + ".f64", g);
    env.grids[a.name] = g;
    if (a.active) {
      sg::DenseGrid gb(shape_of(a, env.sizes));
      read_grid(in_dir + "/" + a.adjoint + ".f64", gb);
      env.grids[a.adjoint] = gb;
    }
  }
  const sg::ArrayDecl& out = sg::output_array(p);
  sg::Env primal = sg::run_nest(p.nest, env);
  write_grid(out_dir + "/primal_" + out.name + ".f64", primal.grids.at(out.name));
  auto prog = sg::assemble_adjoint(p);
  sg::Env gather = sg::run_program(prog, env);
  sg::Env scatter = sg::run_scatter_adjoint(p, env);
  for (const auto& a : p.arrays) {
    if (!a.active || a.name == out.name) continue;
    write_grid(out_dir + "/gather_" + a.adjoint + ".f64", gather.grids.at(a.adjoint));
    write_grid(out_dir + "/scatter_" + a.adjoint + ".f64", scatter.grids.at(a.adjoint));
  }
  return 0;
}

static int cmd_timeloop(const sg::Problem& p, long long n, int T, const std::string& in_dir,
                        const std::string& out_dir, int argc, char** argv) {
  if (T < 2) throw sg::Error("timeloop needs T >= 2");
  std::map<std::string, long long> sz{{"n", n}};
  const sg::ArrayDecl& out = sg::output_array(p);
  const std::string seed = out.adjoint;
  const sg::ArrayDecl* u1d = sg::find_array(p, "u_1");
  const sg::ArrayDecl* u2d = sg::find_array(p, "u_2");
  const sg::ArrayDecl* cd = sg::find_array(p, "c");
  if (!u1d || !u2d || !cd || !u2d->active || !u1d->active || !cd->active)
    throw sg::Error("timeloop: c, u_1, u_2 must be active arrays");
  const auto shape = shape_of(*u1d, sz);
  sg::Env base;
  base.sizes = sz;
  for (const auto& s : p.scalars) base.scalars[s] = 0.0;
  for (int a = 0; a < argc; a++) {
    std::string kv = argv[a];
    auto eq = kv.find('=');
    base.scalars[kv.substr(0, eq)] = std::strtod(kv.c_str() + eq + 1, nullptr);
  }
  sg::DenseGrid c(shape), w(shape);
  read_grid(in_dir + "/c.f64", c);
  read_grid(in_dir + "/w.f64", w);
  std::vector<sg::DenseGrid> u(T + 1, sg::DenseGrid(shape));
  read_grid(in_dir + "/u0.f64", u[0]);
  read_grid(in_dir + "/u1.f64", u[1]);
  // forward: u^{t+1} = run_nest(primal)(c, u_1 = u^t, u_2 = u^{t-1}), u zero-initialised
  for (int t = 1; t < T; t++) {
    sg::Env e = base;
    e.grids["c"] = c;
    e.grids["u_1"] = u[t];
    e.grids["u_2"] = u[t - 1];
    e.grids[out.name] = sg::DenseGrid(shape);
    u[t + 1] = sg::run_nest(p.nest, e).grids.at(out.name);
  }
  // reverse: seed u-bar^{t+1}; accumulate u-bar^t (u_1_b), u-bar^{t-1} (u_2_b), c_b
  const auto prog = sg::assemble_adjoint(p);
  std::vector<sg::DenseGrid> ub(T + 1, sg::DenseGrid(shape));
  ub[T] = w;
  sg::DenseGrid cb(shape);
  for (int t = T - 1; t >= 1; t--) {
    sg::Env e = base;
    e.grids["c"] = c;
    e.grids["u_1"] = u[t];
    e.grids["u_2"] = u[t - 1];
    e.grids[out.name] = sg::DenseGrid(shape);
    e.grids[seed] = ub[t + 1];
    e.grids[u1d->adjoint] = ub[t];
    e.grids[u2d->adjoint] = ub[t - 1];
    e.grids[cd->adjoint] = cb;
    sg::Env r = sg::run_program(prog, e);
    ub[t] = r.grids.at(u1d->adjoint);
    ub[t - 1] = r.grids.at(u2d->adjoint);
    cb = r.grids.at(cd->adjoint);
  }
  write_grid(out_dir + "/u0_b.f64", ub[0]);
  write_grid(out_dir + "/u1_b.f64", ub[1]);
  write_grid(out_dir + "/c_b.f64", cb);
  write_grid(out_dir + "/uT.f64", u[T]);
  return 0;
}

static int cmd_verify(const sg::Problem& p, long long n, unsigned long long seed, int trials) {
  auto rep = sg::verify_problem(p, {{"n", n}}, seed, trials, true);
  std::cout << rep.json_text();
  return rep.pass() ? 0 : 1;
}

// Digest of a grid: element count, sum, sum of squares, first / middle / last
// value, all at full precision (the same function sits in tests/cpp/
// test_host_api.cpp for sgb::make_env).
static void env_digest(std::ostream& os, const std::map<std::string, double>& scalars,
                       const std::map<std::string, std::vector<double>>& grids) {
  char buf[64];
  auto num = [&](double v) {
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    return std::string(buf);
  };
  os << "{\"scalars\":{";
  bool first = true;
  for (const auto& kv : scalars) {
    os << (first ? "" : ",") << "\"" << kv.first << "\":" << num(kv.second);
    first = false;
  }
  os << "},\"grids\":{";
  first = true;
  for (const auto& kv : grids) {
    const std::vector<double>& d = kv.second;
    double s = 0, q = 0;
    for (double x : d) s += x, q += x * x;
    os << (first ? "" : ",") << "\"" << kv.first << "\":[" << d.size() << "," << num(s) << ","
       << num(q) << "," << num(d.empty() ? 0 : d.front()) << ","
       << num(d.empty() ? 0 : d[d.size() / 2]) << "," << num(d.empty() ? 0 : d.back()) << "]";
    first = false;
  }
  os << "}}\n";
}

static int cmd_makeenv(const sg::Problem& p, long long n, unsigned long long seed) {
  const sg::Env env = sg::make_env(p, {{"n", n}}, seed);
  std::map<std::string, std::vector<double>> grids;
  for (const auto& kv : env.grids) grids[kv.first] = kv.second.data();
  env_digest(std::cout, env.scalars, grids);
  return 0;
}

static int cmd_emit(const sg::Problem& p, const std::string& out_dir) {
  sg::EmitOptions opts;
  opts.restrict_pointers = true;  // as cmd_bench (tools/stencilgrad.cpp:286)
  for (const char* fn : {"f", "f_d_a", "f_d_b"})
    opts.opaque_prototypes[fn] = std::string("double ") + fn + "(double a, double b)";
  for (const char* fn : {"g", "g_d_x", "g_d_y"})
    opts.opaque_prototypes[fn] = std::string("double ") + fn + "(double x, double y)";
  auto prog = sg::assemble_adjoint(p);
  std::ofstream(out_dir + "/" + p.name + "_primal.c") << sg::emit_primal(p, opts);
  std::ofstream(out_dir + "/" + p.name + "_adjoint.c") << sg::emit_adjoint(p, prog, opts);
  std::ofstream(out_dir + "/" + p.name + "_scatter.c") << sg::emit_scatter_adjoint(p, opts);
  std::ofstream(out_dir + "/" + p.name + "_protos.h")
      << sg::primal_prototype(p, opts) << sg::adjoint_prototype(p, prog, opts)
      << sg::scatter_prototype(p, opts);
  return 0;
}

int main(int argc, char** argv) {
  try {
    if (argc < 3) {
      std::cerr << "usage: ref_harness info|run|verify|emit <spec> ...\n";
      return 2;
    }
    std::string cmd = argv[1];
    sg::Problem p = load(argv[2]);
    if (cmd == "info" && argc >= 4) return cmd_info(p, std::atoll(argv[3]));
    if (cmd == "run" && argc >= 6)
      return cmd_run(p, std::atoll(argv[3]), argv[4], argv[5], argc - 6, argv + 6);
    if (cmd == "verify" && argc >= 6)
      return cmd_verify(p, std::atoll(argv[3]), std::strtoull(argv[4], nullptr, 10),
                        std::atoi(argv[5]));
    if (cmd == "makeenv" && argc >= 5)
      return cmd_makeenv(p, std::atoll(argv[3]), std::strtoull(argv[4], nullptr, 10));
    if (cmd == "emit" && argc >= 4) return cmd_emit(p, argv[3]);
    if (cmd == "spec") {
      std::cout << sg::serialize_spec(p);
      return 0;
    }
    if (cmd == "b200" && argc >= 5) return cmd_b200(p, std::atoll(argv[3]), argv[4], argc - 5, argv + 5);
    if (cmd == "timeloop" && argc >= 7)
      return cmd_timeloop(p, std::atoll(argv[3]), std::atoi(argv[4]), argv[5], argv[6], argc - 7,
                          argv + 7);
    if (cmd == "canon") {
      std::cout << sg::b200_program_text(sg::assemble_adjoint(p));
      return 0;
    }
    if (cmd == "match") {
      std::string why;
      const std::string fam = sg::b200_program_family(sg::assemble_adjoint(p), &why);
      for (auto& ch : why)
        if (ch == '"' || ch == '\\' || ch == '\n') ch = ' ';
      std::cout << "{\"name\":\"" << p.name << "\",\"family\":"
                << (fam.empty() ? std::string("null") : "\"" + fam + "\"")
                << ",\"why\":\"" << why << "\"}\n";
      return 0;
    }
    std::cerr << "bad arguments\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
