// Host-buffer entry point: the reference-facing call with HOST arrays.
//
// Mirrors the emitted CPU function (a caller hands host arrays to <name>_b
// and gets the accumulated adjoints back, codegen.cpp:332-382) on the B200:
// H2D of every referenced array (the adjoints too -- the contract is +=),
// the gather-adjoint launch, D2H of the accumulated adjoints, then a stream
// synchronisation so the call returns with results in host memory like the
// CPU function does.  The plan owns the device workspace (no allocation in
// the call).  One cudaMemcpyAsync per array (no batched-copy APIs).
#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "sgb_common.cuh"

struct sgb_plan {
  std::string family;
  int n = 0, dtype = 0, dims = 0;
  // z-slab: local planes [i_base, i_base + nplanes), outputs [out_i0, out_i1)
  // (the full grid: 0, n, 0, n)
  int i_base = 0, nplanes = 0, out_i0 = 0, out_i1 = 0;
  size_t bytes = 0;
  std::vector<void*> dev;
  std::vector<bool> rmw;  // accumulated adjoint arrays (copied back)
  // 3D families: copies and compute pipelined over i-chunks on three streams
  cudaStream_t s_h2d = nullptr, s_cmp = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_in, ev_out;
  int chunks = 1;
  bool in_sweep = false;  // c, c_b resident (sgb_plan_sweep_*)
};

namespace {

struct FamSpec {
  const char* name;
  int dims;
  int narr;
  bool rmw[6];
};

const FamSpec kFams[] = {
    // wave1d_b(n, D, c, c_b, u, u_b, u_prev_b, u_next_b)
    {"wave1d", 1, 6, {false, true, false, true, true, false}},
    // wave3d_c_b(n, D, c, c_b, u_1, u_1_b, u_2_b, u_b)
    {"wave3d_c", 3, 6, {false, true, false, true, true, false}},
    {"wave3d_c2", 3, 6, {false, true, false, true, true, false}},
    // burgers2d_b(n, C, D, u_1, u_1_b, u_b)
    {"burgers2d", 2, 3, {false, true, false}},
    // wave3d_r4_b(n, D, c, c_b, u_1, u_1_b, u_b)
    {"wave3d_r4", 3, 5, {false, true, false, true, false}},
};

const FamSpec* find_fam(const std::string& f) {
  for (const auto& s : kFams)
    if (f == s.name) return &s;
  return nullptr;
}

}  // namespace

extern "C" {

sgb_plan* sgb_plan_create_slab(const char* family, int n, int dtype_bytes, int i_base,
                               int nplanes, int out_i0, int out_i1) {
  const FamSpec* fs = family ? find_fam(family) : nullptr;
  if (!fs || n <= 0 || (dtype_bytes != 4 && dtype_bytes != 8)) {
    sgb::set_error("sgb_plan_create: unsupported family/n/dtype");
    return nullptr;
  }
  const bool full = i_base == 0 && nplanes == n && out_i0 == 0 && out_i1 == n;
  const bool has_slab = std::string(family) == "wave3d_r4" || std::string(family) == "wave3d_c";
  if (!full && (!has_slab || i_base < 0 || nplanes <= 0 ||
                i_base + nplanes > n || out_i0 < i_base || out_i1 > i_base + nplanes ||
                out_i0 >= out_i1)) {
    sgb::set_error("sgb_plan_create_slab: slabs need wave3d_r4 / wave3d_c and "
                   "i_base <= out_i0 < out_i1 <= i_base + nplanes <= n");
    return nullptr;
  }
  auto* p = new sgb_plan;
  p->family = family;
  p->n = n;
  p->dtype = dtype_bytes;
  p->dims = fs->dims;
  p->i_base = i_base;
  p->nplanes = nplanes;
  p->out_i0 = out_i0;
  p->out_i1 = out_i1;
  size_t elems = 1;
  for (int d = 0; d < fs->dims - 1; d++) elems *= (size_t)n;
  elems *= (size_t)(fs->dims == 3 ? nplanes : n);
  p->bytes = elems * dtype_bytes;
  for (int a = 0; a < fs->narr; a++) {
    void* d = nullptr;
    if (cudaMalloc(&d, p->bytes) != cudaSuccess) {
      sgb::set_error("sgb_plan_create: cudaMalloc failed");
      for (void* q : p->dev) cudaFree(q);
      delete p;
      return nullptr;
    }
    p->dev.push_back(d);
    p->rmw.push_back(fs->rmw[a]);
  }
  // pipelined host path (3D fp32 slabs / grids, burgers2d rows, wave1d index
  // ranges, on the shapes the range kernels take): C chunks of the outermost
  // dimension; the call costs ~ H2D(all) + D2H(one chunk), so more chunks
  // shorten the tail
  const long long units = fs->dims == 3 ? nplanes : n;  // planes / rows / elements
  const bool pipelined = (fs->dims == 3 && p->family != "wave3d_c2") ||
                         (fs->dims == 2 && ((long long)n * dtype_bytes) % 16 == 0) ||
                         (fs->dims == 1 && n % 2 == 0);
  if (pipelined) {
    // 3D: ~16-plane chunks (at most 64): 1024^3 e2e 425 -> 421 ms for 32 -> 64
    // chunks, 0.98-0.99 of the box's concurrent-copy floor (scripts/e2e_time.py)
    int c = units >= 128 ? 32 : 1;
    if (fs->dims == 3 && units >= 128) c = (int)std::min<long long>(64, units / 16);
    if (sgb::opt(sgb::OPT_PLAN_CHUNKS, 0) > 0) c = (int)sgb::opt(sgb::OPT_PLAN_CHUNKS, 0);
    p->chunks = (int)std::min<long long>(c, std::max<long long>(1, units / 16));
    cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&p->s_cmp, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking);
    p->ev_in.resize(p->chunks);
    p->ev_out.resize(p->chunks);
    for (int k = 0; k < p->chunks; k++) {
      cudaEventCreateWithFlags(&p->ev_in[k], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&p->ev_out[k], cudaEventDisableTiming);
    }
  }
  return p;
}

sgb_plan* sgb_plan_create(const char* family, int n, int dtype_bytes) {
  return sgb_plan_create_slab(family, n, dtype_bytes, 0, n, 0, n);
}

void sgb_plan_destroy(sgb_plan* plan) {
  if (!plan) return;
  for (void* d : plan->dev) cudaFree(d);
  for (auto e : plan->ev_in) cudaEventDestroy(e);
  for (auto e : plan->ev_out) cudaEventDestroy(e);
  if (plan->s_h2d) cudaStreamDestroy(plan->s_h2d);
  if (plan->s_cmp) cudaStreamDestroy(plan->s_cmp);
  if (plan->s_d2h) cudaStreamDestroy(plan->s_d2h);
  delete plan;
}

// Chunked families: H2D of chunk c+1 (copy engine), the adjoint of chunk c's
// outputs (SMs) and D2H of chunk c-1 (other copy engine) overlap.  The
// outermost dimension (3D: local planes, 2D: rows, 1D: elements) is split
// into C chunks; the outputs inside chunk c need inputs up to R = 1..4 units
// beyond it, so chunk c's kernel waits for the H2D of chunks c and c+1.
// `up` / `down`: which arrays are copied in / out (a reverse sweep keeps c and
// c_b resident and moves only the step's states and adjoint); `fresh`: the
// radius-4 gather writes u_1_b as the step's adjoint alone.
static int run_pipelined(sgb_plan* p, const double* scalars, void** arrays,
                         const std::vector<bool>& up, const std::vector<bool>& down,
                         bool fresh) {
  const int n = p->n, C = p->chunks, base = p->i_base;
  const int L = p->dims == 3 ? p->nplanes : n;
  // bytes of one unit of the outermost dimension
  const size_t plane = (size_t)(p->dims == 3 ? (long long)n * n : (p->dims == 2 ? n : 1)) *
                       p->dtype;
  auto bound = [&](int c) {  // local unit; 1D chunk bounds even (2-point threads)
    const long long b = (long long)L * c / C;
    return (int)(p->dims == 1 ? b & ~1LL : b);
  };
  const size_t na = p->dev.size();
  for (int c = 0; c < C; c++) {
    const int a = bound(c), b = bound(c + 1);
    for (size_t k = 0; k < na; k++) {
      if (!up[k]) continue;
      if (cudaMemcpyAsync((char*)p->dev[k] + a * plane, (const char*)arrays[k] + a * plane,
                          (b - a) * plane, cudaMemcpyHostToDevice, p->s_h2d) != cudaSuccess) {
        sgb::set_error("sgb_plan_run_adjoint_host: H2D copy failed");
        return -1;
      }
    }
    cudaEventRecord(p->ev_in[c], p->s_h2d);
  }
  for (int c = 0; c < C; c++) {
    // output planes of this chunk (global indices)
    const int a = std::max(p->out_i0, base + bound(c));
    const int b = std::min(p->out_i1, base + bound(c + 1));
    cudaStreamWaitEvent(p->s_cmp, p->ev_in[c], 0);
    if (c + 1 < C) cudaStreamWaitEvent(p->s_cmp, p->ev_in[c + 1], 0);
    if (a < b) {
      int rc = SGB_EINVAL;
      if (p->dims == 3 && p->dtype == 4) {
        float** d = reinterpret_cast<float**>(p->dev.data());
        if (p->family == "wave3d_r4")
          rc = fresh ? wave3d_r4_b_fresh_slab_f32(n, scalars[0], d[0], d[1], d[2], d[3], d[4],
                                                  base, L, a, b, p->s_cmp)
                     : wave3d_r4_b_slab_f32(n, scalars[0], d[0], d[1], d[2], d[3], d[4], base, L,
                                            a, b, p->s_cmp);
        else if (p->family == "wave3d_c")
          rc = wave3d_c_b_slab_f32(n, scalars[0], d[0], d[1], d[2], d[3], d[4], d[5], base, L,
                                   a, b, p->s_cmp);
      } else if (p->dims == 3) {
        double** d = reinterpret_cast<double**>(p->dev.data());
        if (p->family == "wave3d_r4")
          rc = fresh ? wave3d_r4_b_fresh_slab_f64(n, scalars[0], d[0], d[1], d[2], d[3], d[4],
                                                  base, L, a, b, p->s_cmp)
                     : wave3d_r4_b_slab_f64(n, scalars[0], d[0], d[1], d[2], d[3], d[4], base, L,
                                            a, b, p->s_cmp);
        else if (p->family == "wave3d_c")
          rc = wave3d_c_b_slab_f64(n, scalars[0], d[0], d[1], d[2], d[3], d[4], d[5], base, L,
                                   a, b, p->s_cmp);
      } else if (p->dtype == 8) {
        double** d = reinterpret_cast<double**>(p->dev.data());
        if (p->family == "burgers2d")
          rc = burgers2d_b_rows_f64(n, scalars[0], scalars[1], d[0], d[1], d[2], a, b, p->s_cmp);
        else if (p->family == "wave1d")
          rc = wave1d_b_range_f64(n, scalars[0], d[0], d[1], d[2], d[3], d[4], d[5], a, b,
                                  p->s_cmp);
      } else {
        float** d = reinterpret_cast<float**>(p->dev.data());
        if (p->family == "burgers2d")
          rc = burgers2d_b_rows_f32(n, scalars[0], scalars[1], d[0], d[1], d[2], a, b, p->s_cmp);
        else if (p->family == "wave1d")
          rc = wave1d_b_range_f32(n, scalars[0], d[0], d[1], d[2], d[3], d[4], d[5], a, b,
                                  p->s_cmp);
      }
      if (rc != 0) return rc;
    }
    cudaEventRecord(p->ev_out[c], p->s_cmp);
    cudaStreamWaitEvent(p->s_d2h, p->ev_out[c], 0);
    if (a >= b) continue;
    const size_t off = (size_t)(a - base) * plane, len = (size_t)(b - a) * plane;
    for (size_t k = 0; k < na; k++) {
      if (!down[k]) continue;
      if (cudaMemcpyAsync((char*)arrays[k] + off, (const char*)p->dev[k] + off, len,
                          cudaMemcpyDeviceToHost, p->s_d2h) != cudaSuccess) {
        sgb::set_error("sgb_plan_run_adjoint_host: D2H copy failed");
        return -1;
      }
    }
  }
  if (cudaStreamSynchronize(p->s_d2h) != cudaSuccess) {
    sgb::set_error("sgb_plan_run_adjoint_host: stream synchronisation failed");
    return -1;
  }
  return 0;
}

int sgb_plan_run_adjoint_host(sgb_plan* p, const double* scalars, void** arrays,
                              sgb_stream_t stream) {
  if (!p || !arrays || !scalars) {
    sgb::set_error("sgb_plan_run_adjoint_host: null argument");
    return SGB_EINVAL;
  }
  if (p->in_sweep) {  // the call would overwrite the sweep's resident arrays
    sgb::set_error("sgb_plan_run_adjoint_host: a sweep is open on this plan (sgb_plan_sweep_end)");
    return SGB_EINVAL;
  }
  if (p->s_cmp) {
    for (size_t a = 0; a < p->dev.size(); a++)
      if (!arrays[a]) {
        sgb::set_error("sgb_plan_run_adjoint_host: null host array");
        return SGB_EINVAL;
      }
    // order the pipeline after the caller's stream, then run on our streams
    cudaEvent_t start;
    cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    cudaEventRecord(start, sgb::as_stream(stream));
    cudaStreamWaitEvent(p->s_h2d, start, 0);
    cudaEventDestroy(start);
    return run_pipelined(p, scalars, arrays, std::vector<bool>(p->dev.size(), true), p->rmw,
                         false);
  }
  cudaStream_t s = sgb::as_stream(stream);
  const size_t na = p->dev.size();
  for (size_t a = 0; a < na; a++) {
    if (!arrays[a]) {
      sgb::set_error("sgb_plan_run_adjoint_host: null host array");
      return SGB_EINVAL;
    }
    if (cudaMemcpyAsync(p->dev[a], arrays[a], p->bytes, cudaMemcpyHostToDevice, s) !=
        cudaSuccess) {
      sgb::set_error("sgb_plan_run_adjoint_host: H2D copy failed");
      return -1;
    }
  }
  int rc = SGB_EINVAL;
  void** d = p->dev.data();
  const std::string& f = p->family;
  if (p->dtype == 4) {
    float** a = reinterpret_cast<float**>(d);
    if (f == "wave1d") rc = wave1d_b_f32(p->n, scalars[0], a[0], a[1], a[2], a[3], a[4], a[5], stream);
    if (f == "wave3d_c") rc = wave3d_c_b_f32(p->n, scalars[0], a[0], a[1], a[2], a[3], a[4], a[5], stream);
    if (f == "wave3d_c2") rc = wave3d_c2_b_f32(p->n, scalars[0], a[0], a[1], a[2], a[3], a[4], a[5], stream);
    if (f == "burgers2d") rc = burgers2d_b_f32(p->n, scalars[0], scalars[1], a[0], a[1], a[2], stream);
    if (f == "wave3d_r4") rc = wave3d_r4_b_f32(p->n, scalars[0], a[0], a[1], a[2], a[3], a[4], stream);
  } else {
    double** a = reinterpret_cast<double**>(d);
    if (f == "wave1d") rc = wave1d_b_f64(p->n, scalars[0], a[0], a[1], a[2], a[3], a[4], a[5], stream);
    if (f == "wave3d_c") rc = wave3d_c_b_f64(p->n, scalars[0], a[0], a[1], a[2], a[3], a[4], a[5], stream);
    if (f == "wave3d_c2") rc = wave3d_c2_b_f64(p->n, scalars[0], a[0], a[1], a[2], a[3], a[4], a[5], stream);
    if (f == "burgers2d") rc = burgers2d_b_f64(p->n, scalars[0], scalars[1], a[0], a[1], a[2], stream);
    if (f == "wave3d_r4") rc = wave3d_r4_b_f64(p->n, scalars[0], a[0], a[1], a[2], a[3], a[4], stream);
  }
  if (rc != 0) return rc;
  for (size_t a = 0; a < na; a++) {
    if (!p->rmw[a]) continue;
    if (cudaMemcpyAsync(arrays[a], p->dev[a], p->bytes, cudaMemcpyDeviceToHost, s) !=
        cudaSuccess) {
      sgb::set_error("sgb_plan_run_adjoint_host: D2H copy failed");
      return -1;
    }
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    sgb::set_error("sgb_plan_run_adjoint_host: stream synchronisation failed");
    return -1;
  }
  return 0;
}

// ---- reverse sweeps over host-held states -----------------------------------
// The multi-step BASELINE protocols with the forward states checkpointed in
// host memory.  Whatever does not change per step stays RESIDENT on the device
// between sweep_begin and sweep_end.
//   wave3d_r4 (cfg 5: independent steps; c, c_b, u_1, u_1_b, u_b): c and the
//     accumulator c_b resident; a step moves u_1 and u_b in and the step's own
//     adjoint u_1_b out (8 + 4 bytes per point in fp32 against the 20 + 8 of the
//     accumulating call).
//   wave3d_c (cfg 2: carried steps; c, c_b, u_1, u_1_b, u_2_b, u_b):
//     c, c_b and the three adjoints resident; a step moves only the state u_1
//     in, accumulates, and rotates the adjoints on the device (seed <- u_1_b,
//     u_1_b <- u_2_b, u_2_b <- 0) -- 4 bytes per point per step instead of
//     24 + 12; sweep_end returns c_b, u_1_b, u_2_b and the seed u_b.
namespace {

struct SweepSpec {
  const char* family;
  std::vector<bool> begin_up, step_up, step_down, end_down;
  bool fresh, carried;
};

const SweepSpec* sweep_spec(const std::string& fam) {
  static const SweepSpec specs[] = {
      {"wave3d_r4", {1, 1, 0, 0, 0}, {0, 0, 1, 0, 1}, {0, 0, 0, 1, 0}, {0, 1, 0, 0, 0}, true,
       false},
      {"wave3d_c", {1, 1, 0, 1, 1, 1}, {0, 0, 1, 0, 0, 0}, {0, 0, 0, 0, 0, 0},
       {0, 1, 0, 1, 1, 1}, false, true},
  };
  for (const auto& sp : specs)
    if (fam == sp.family) return &sp;
  return nullptr;
}

}  // namespace

static const SweepSpec* sweep_check(sgb_plan* p, void** arrays, const char* who) {
  if (!p || !arrays) {
    sgb::set_error(std::string(who) + ": null argument");
    return nullptr;
  }
  const SweepSpec* sp = sweep_spec(p->family);
  const bool full = p->i_base == 0 && p->nplanes == p->n;
  if (!sp || !p->s_cmp || (sp->carried && !full)) {
    sgb::set_error(std::string(who) + ": sweeps need a pipelined wave3d_r4 plan (grid or "
                   "slab) or a full-grid wave3d_c plan");
    return nullptr;
  }
  return sp;
}

static int sweep_copies(sgb_plan* p, void** arrays, const std::vector<bool>& which,
                        cudaMemcpyKind kind, sgb_stream_t stream, const char* who) {
  cudaStream_t s = sgb::as_stream(stream);
  for (size_t k = 0; k < which.size(); k++) {
    if (!which[k]) continue;
    if (!arrays[k]) {
      sgb::set_error(std::string(who) + ": null host array");
      return SGB_EINVAL;
    }
    const cudaError_t e = kind == cudaMemcpyHostToDevice
                              ? cudaMemcpyAsync(p->dev[k], arrays[k], p->bytes, kind, s)
                              : cudaMemcpyAsync(arrays[k], p->dev[k], p->bytes, kind, s);
    if (e != cudaSuccess) {
      sgb::set_error(std::string(who) + ": copy failed");
      return -1;
    }
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    sgb::set_error(std::string(who) + ": copy failed");
    return -1;
  }
  return 0;
}

int sgb_plan_sweep_begin(sgb_plan* p, void** arrays, sgb_stream_t stream) {
  const SweepSpec* sp = sweep_check(p, arrays, "sgb_plan_sweep_begin");
  if (!sp) return SGB_EINVAL;
  if (int rc = sweep_copies(p, arrays, sp->begin_up, cudaMemcpyHostToDevice, stream,
                            "sgb_plan_sweep_begin"))
    return rc;
  p->in_sweep = true;
  return 0;
}

int sgb_plan_sweep_step_host(sgb_plan* p, const double* scalars, void** arrays,
                             sgb_stream_t stream) {
  const SweepSpec* sp = sweep_check(p, arrays, "sgb_plan_sweep_step_host");
  if (!sp) return SGB_EINVAL;
  if (!scalars || !p->in_sweep) {
    sgb::set_error("sgb_plan_sweep_step_host: no sweep begun on this plan");
    return SGB_EINVAL;
  }
  for (size_t k = 0; k < sp->step_up.size(); k++)
    if ((sp->step_up[k] || sp->step_down[k]) && !arrays[k]) {
      sgb::set_error("sgb_plan_sweep_step_host: null host array");
      return SGB_EINVAL;
    }
  cudaEvent_t start;
  cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  cudaEventRecord(start, sgb::as_stream(stream));
  cudaStreamWaitEvent(p->s_h2d, start, 0);
  cudaEventDestroy(start);
  if (int rc = run_pipelined(p, scalars, arrays, sp->step_up, sp->step_down, sp->fresh))
    return rc;
  if (sp->carried) {
    // every chunk's gather is complete (run_pipelined waited for them): rotate
    // seed <- u_1_b, u_1_b <- u_2_b, u_2_b <- the old seed's buffer, zeroed
    void* seed = p->dev[5];
    p->dev[5] = p->dev[3];
    p->dev[3] = p->dev[4];
    p->dev[4] = seed;
    if (cudaMemsetAsync(p->dev[4], 0, p->bytes, p->s_cmp) != cudaSuccess ||
        cudaStreamSynchronize(p->s_cmp) != cudaSuccess) {
      sgb::set_error("sgb_plan_sweep_step_host: rotation failed");
      return -1;
    }
  }
  return 0;
}

int sgb_plan_sweep_end(sgb_plan* p, void** arrays, sgb_stream_t stream) {
  const SweepSpec* sp = sweep_check(p, arrays, "sgb_plan_sweep_end");
  if (!sp) return SGB_EINVAL;
  if (!p->in_sweep) {
    sgb::set_error("sgb_plan_sweep_end: no sweep begun on this plan");
    return SGB_EINVAL;
  }
  p->in_sweep = false;
  return sweep_copies(p, arrays, sp->end_down, cudaMemcpyDeviceToHost, stream,
                      "sgb_plan_sweep_end");
}

}  // extern "C"
