// Host-buffer entry point: the reference-facing call with HOST arrays.
//
// Mirrors the emitted CPU function (a caller hands host arrays to <name>_b
// and gets the accumulated adjoints back, codegen.cpp:332-382) on the B200:
// H2D of every referenced array (the adjoints too -- the contract is +=),
// the gather-adjoint launch, D2H of the accumulated adjoints, then a stream
// synchronisation so the call returns with results in host memory like the
// CPU function does.  The plan owns the device workspace (no allocation in
// the call).  One cudaMemcpyAsync per array (no batched-copy APIs).
#include <string>
#include <vector>

#include "sgb_common.cuh"

struct sgb_plan {
  std::string family;
  int n = 0, dtype = 0, dims = 0;
  size_t bytes = 0;
  std::vector<void*> dev;
  std::vector<bool> rmw;  // accumulated adjoint arrays (copied back)
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

sgb_plan* sgb_plan_create(const char* family, int n, int dtype_bytes) {
  const FamSpec* fs = family ? find_fam(family) : nullptr;
  if (!fs || n <= 0 || (dtype_bytes != 4 && dtype_bytes != 8)) {
    sgb::set_error("sgb_plan_create: unsupported family/n/dtype");
    return nullptr;
  }
  auto* p = new sgb_plan;
  p->family = family;
  p->n = n;
  p->dtype = dtype_bytes;
  p->dims = fs->dims;
  size_t elems = 1;
  for (int d = 0; d < fs->dims; d++) elems *= (size_t)n;
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
  return p;
}

void sgb_plan_destroy(sgb_plan* plan) {
  if (!plan) return;
  for (void* d : plan->dev) cudaFree(d);
  delete plan;
}

int sgb_plan_run_adjoint_host(sgb_plan* p, const double* scalars, void** arrays,
                              sgb_stream_t stream) {
  if (!p || !arrays || !scalars) {
    sgb::set_error("sgb_plan_run_adjoint_host: null argument");
    return SGB_EINVAL;
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

}  // extern "C"
