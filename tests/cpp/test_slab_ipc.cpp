// Multi-GPU z-slab plan (sgb_slab_*, include/stencilgrad_b200.h) driven from
// C++ with the IPC copy-engine transport: W processes (fork()ed before any
// CUDA call) on ONE GPU, each a rank of a z-slab decomposition of a wave3d_r4
// grid.  Blobs go through pipes (the out-of-band channel a solver would use:
// MPI, a file, torch.distributed).  Every rank runs T reverse steps of cfg 5's
// protocol -- u_1 / u_b regenerated from (seed, step) on its OWNED planes
// only, halos NaN-poisoned and refreshed by the plan's exchange, u_1_b fresh
// per step, c_b accumulated -- in three schedules (exchange then compute,
// interior overlapped with the exchange, and the exchange of step t+1
// pipelined behind step t on a second buffer set), and compares its owned
// planes with the single-GPU full-grid result it computes itself: bitwise.
// No kernel waits on another process: ordering is stream memory operations
// on the plan's comm stream.  Built and run by tests/test_slab_plan.py.
#include <sys/wait.h>
#include <unistd.h>

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "stencilgrad_b200.h"

#define CK(x)                                                                     \
  do {                                                                            \
    auto rc_ = (x);                                                               \
    if (rc_ != 0) {                                                               \
      std::fprintf(stderr, "rank %d: %s failed (%d): %s\n", g_rank, #x, (int)rc_, \
                   sgb_last_error());                                             \
      std::exit(3);                                                               \
    }                                                                             \
  } while (0)

static int g_rank = -1;

static bool write_all(int fd, const void* p, size_t n) {
  const char* c = static_cast<const char*>(p);
  while (n) {
    const ssize_t k = write(fd, c, n);
    if (k <= 0) return false;
    c += k;
    n -= (size_t)k;
  }
  return true;
}
static bool read_all(int fd, void* p, size_t n) {
  char* c = static_cast<char*>(p);
  while (n) {
    const ssize_t k = read(fd, c, n);
    if (k <= 0) return false;
    c += k;
    n -= (size_t)k;
  }
  return true;
}

// regenerate step t's u_1 / u_b on global planes [i0, i0 + np) of a local array
// whose first plane is global plane `base` (counter-based: same values in
// every decomposition; drivers.regen_state / regen_seed)
static void regen(float* u1, float* ub, int n, int base, int i0, int np, int t,
                  cudaStream_t s) {
  const size_t plane = (size_t)n * n;
  CK(sgb_fill_normal3d_f32(u1 + (size_t)(i0 - base) * plane, n, i0, np, 4, 0, 1000 + 2 * t, 0.0,
                           1.0, s));
  CK(sgb_fill_normal3d_f32(ub + (size_t)(i0 - base) * plane, n, i0, np, 0, 0, 1001 + 2 * t, 0.0,
                           1.0, s));
}

static int run_rank(int rank, int world, int n, int T, int to_parent, int from_parent) {
  g_rank = rank;
  CK(cudaSetDevice(0));
  const double D = 0.01;
  const size_t plane = (size_t)n * n, full = plane * n;
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));

  // ---- single-GPU reference on the full grid
  float *c, *cb, *u1, *u1b, *ub;
  for (float** p : {&c, &cb, &u1, &u1b, &ub}) CK(cudaMalloc(p, full * sizeof(float)));
  CK(sgb_fill_layered_f32(c, n, 8, 1.5, 4.5, 0, 0, n, s));
  CK(cudaMemsetAsync(cb, 0, full * sizeof(float), s));
  for (int t = 0; t < T; t++) {
    regen(u1, ub, n, 0, 0, n, t, s);
    CK(wave3d_r4_b_fresh_f32(n, D, c, cb, u1, u1b, ub, s));
  }
  std::vector<float> ref_cb(full), ref_u1b(full);
  CK(cudaMemcpyAsync(ref_cb.data(), cb, full * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(ref_u1b.data(), u1b, full * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (float* p : {c, cb, u1, u1b, ub}) CK(cudaFree(p));

  // ---- this rank's slab
  sgb_slab* plan = sgb_slab_create("wave3d_r4", n, 4, rank, world, SGB_TRANSPORT_IPC, nullptr);
  if (!plan) {
    std::fprintf(stderr, "rank %d: sgb_slab_create: %s\n", rank, sgb_last_error());
    return 3;
  }
  int base, np, own0, own1;
  CK(sgb_slab_geometry(plan, &base, &np, &own0, &own1));
  const size_t local = plane * np;
  float *lc, *lcb, *lu1b, *lu1[2], *lub[2];
  for (float** p : {&lc, &lcb, &lu1b, &lu1[0], &lu1[1], &lub[0], &lub[1]})
    CK(cudaMalloc(p, local * sizeof(float)));
  // NaN everywhere (halos must come from the exchange), then the owned planes
  std::vector<float> nan(local, std::nanf(""));
  for (float* p : {lc, lu1[0], lu1[1], lub[0], lub[1]})
    CK(cudaMemcpy(p, nan.data(), local * 4, cudaMemcpyHostToDevice));
  CK(sgb_fill_layered_f32(lc + (size_t)(own0 - base) * plane, n, 8, 1.5, 4.5, 0, own0,
                          own1 - own0, s));
  CK(sgb_slab_bind(plan, 0, "c", lc));
  CK(sgb_slab_bind(plan, 0, "c_b", lcb));
  CK(sgb_slab_bind(plan, 0, "u_1_b", lu1b));
  for (int k = 0; k < 2; k++) {
    CK(sgb_slab_bind(plan, k, "u_1", lu1[k]));
    CK(sgb_slab_bind(plan, k, "u_b", lub[k]));
  }
  long long bytes = 0;
  CK(sgb_slab_ipc_export(plan, nullptr, &bytes));
  std::vector<char> mine(bytes), all(bytes * world);
  CK(sgb_slab_ipc_export(plan, mine.data(), &bytes));
  CK(cudaDeviceSynchronize());
  if (!write_all(to_parent, &bytes, sizeof(bytes)) || !write_all(to_parent, mine.data(), bytes) ||
      !read_all(from_parent, all.data(), all.size()))
    return 4;
  CK(sgb_slab_ipc_connect(plan, rank > 0 ? &all[(rank - 1) * bytes] : nullptr,
                          rank < world - 1 ? &all[(rank + 1) * bytes] : nullptr));
  // connection probe: every rank's phase 0 before anyone's phase 1
  char sync = 1;
  CK(sgb_slab_ipc_probe(plan, 0));
  if (!write_all(to_parent, &sync, 1) || !read_all(from_parent, &sync, 1)) return 4;
  CK(sgb_slab_ipc_probe(plan, 1));
  CK(sgb_slab_halo_start(plan, 0, 1u, s));  // c is static: its halo once

  const double sc[1] = {D};
  int bad = 0;
  const char* names[3] = {"exchange_then_compute", "overlapped", "pipelined"};
  for (int mode = 0; mode < 3; mode++) {
    CK(cudaMemsetAsync(lcb, 0, local * 4, s));
    if (mode < 2) {
      for (int t = 0; t < T; t++) {
        regen(lu1[0], lub[0], n, base, own0, own1 - own0, t, s);
        CK(sgb_slab_step(plan, 0, sc, SGB_STEP_FRESH | (mode == 1 ? SGB_STEP_OVERLAP : 0), s));
      }
    } else {
      // step t reads set t % 2; step t+1's regeneration + exchange is queued
      // before step t's compute (same stream here, comm stream for the copies)
      regen(lu1[0], lub[0], n, base, own0, own1 - own0, 0, s);
      CK(sgb_slab_halo_start(plan, 0, 2u | 4u, s));
      for (int t = 0; t < T; t++) {
        if (t + 1 < T) {
          const int k = (t + 1) % 2;
          regen(lu1[k], lub[k], n, base, own0, own1 - own0, t + 1, s);
          CK(sgb_slab_halo_start(plan, k, 2u | 4u, s));
        }
        CK(sgb_slab_step(plan, t % 2, sc, SGB_STEP_FRESH | SGB_STEP_NO_EXCHANGE, s));
      }
    }
    CK(cudaStreamSynchronize(s));
    std::vector<float> got(local);
    for (int which = 0; which < 2; which++) {
      CK(cudaMemcpy(got.data(), which ? lu1b : lcb, local * 4, cudaMemcpyDeviceToHost));
      const std::vector<float>& want = which ? ref_u1b : ref_cb;
      const size_t a = (size_t)(own0 - base) * plane, cnt = (size_t)(own1 - own0) * plane;
      if (std::memcmp(got.data() + a, want.data() + (size_t)own0 * plane, cnt * 4) != 0) {
        std::fprintf(stderr, "rank %d %s: %s differs from the single-GPU result\n", rank,
                     names[mode], which ? "u_1_b" : "c_b");
        bad++;
      }
    }
  }
  // nobody unmaps / frees before every rank is done with its neighbours'
  // memory: one more round through the parent
  char tok = 1;
  if (!write_all(to_parent, &tok, 1) || !read_all(from_parent, &tok, 1)) return 4;
  sgb_slab_destroy(plan);
  for (float* p : {lc, lcb, lu1b, lu1[0], lu1[1], lub[0], lub[1]}) cudaFree(p);
  std::printf("rank %d: owned planes [%d, %d) %s\n", rank, own0, own1, bad ? "FAIL" : "ok");
  return bad ? 1 : 0;
}

int main(int argc, char** argv) {
  const int world = argc > 1 ? std::atoi(argv[1]) : 2;
  const int n = argc > 2 ? std::atoi(argv[2]) : 72;
  const int T = argc > 3 ? std::atoi(argv[3]) : 4;
  std::vector<int> up(world), down(world), pid(world);
  for (int r = 0; r < world; r++) {
    int a[2], b[2];
    if (pipe(a) || pipe(b)) return 2;
    const int p = fork();
    if (p == 0) {
      close(a[0]);
      close(b[1]);
      std::exit(run_rank(r, world, n, T, a[1], b[0]));
    }
    close(a[1]);
    close(b[0]);
    up[r] = a[0];
    down[r] = b[1];
    pid[r] = p;
  }
  // gather the blobs, hand every rank all of them; then two barrier rounds
  // (the parent never touches CUDA)
  std::vector<char> all;
  bool ok = true;
  for (int r = 0; r < world && ok; r++) {
    long long bytes = 0;
    ok = read_all(up[r], &bytes, sizeof(bytes)) && bytes > 0 && bytes < (1 << 20);
    if (!ok) break;
    std::vector<char> buf(bytes);
    ok = read_all(up[r], buf.data(), bytes);
    all.insert(all.end(), buf.begin(), buf.end());
  }
  for (int r = 0; r < world && ok; r++) ok = write_all(down[r], all.data(), all.size());
  char tok;
  for (int round = 0; round < 2; round++) {  // the probe barrier, then the final one
    for (int r = 0; r < world && ok; r++) ok = read_all(up[r], &tok, 1);
    for (int r = 0; r < world && ok; r++) ok = write_all(down[r], &tok, 1);
  }
  int failures = ok ? 0 : 1;
  for (int r = 0; r < world; r++) {
    int st = 0;
    waitpid(pid[r], &st, 0);
    if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) failures++;
  }
  std::printf("slab_ipc: world %d n %d steps %d: %s\n", world, n, T, failures ? "FAIL" : "ok");
  return failures ? 1 : 0;
}
