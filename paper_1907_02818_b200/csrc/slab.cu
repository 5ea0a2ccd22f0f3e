// Multi-GPU z-slab plan: one rank per GPU owns the global planes
// [own0, own1) of the outermost counter i and holds R halo planes on each
// interior side; the gather form writes only owned planes, so the single
// exchange per reverse step is the forward halo of the fields read at an
// i-offset (u_1 and the seed u_b; c once, it is static).  The plan owns the
// communication -- an NCCL communicator or a CUDA-IPC copy-engine transport --
// and a comm stream; the caller owns every array (the reference ABI's
// contract, codegen.cpp:213-230) and binds them once.
//
// Transports
//   SGB_TRANSPORT_NCCL: ncclSend / ncclRecv of the R edge planes to p +- 1 in
//     one ncclGroupStart/End on the comm stream (NVLink / NVSwitch between the
//     GPUs of a box).  libnccl.so.2 is dlopen'ed (the one torch already loaded
//     when present), so the library has no link-time NCCL dependency.
//   SGB_TRANSPORT_IPC: every rank maps its neighbours' arrays and a small flag
//     buffer (CUDA IPC; peer memory over NVLink) and PUSHES its edge planes
//     into their halo planes with one cudaMemcpyAsync per field and side on
//     the comm stream -- copy engines, no SMs, so the exchange overlaps a
//     one-CTA-per-SM gather completely.  Ordering is device-side with stream
//     memory operations on 32-bit epoch flags: a rank tells each neighbour
//     "my halo of set s is free for epoch e" (remote write), waits for the
//     neighbour's same message before pushing, then writes "epoch e arrived"
//     into the neighbour's flags; consumers wait on their own flags.  No host
//     round trip, no kernel that spins.
//
// Double-buffered inputs (set 0 / 1) let a driver pipeline the exchange of
// step t+1 behind the compute of step t (drivers.HaloPrefetch): arrays not
// bound for set 1 fall back to set 0's.
#include <dlfcn.h>

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "sgb_common.cuh"

namespace sgb {
namespace {

// ---------------------------------------------------------------- NCCL (dlopen)
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string err;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) n.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) {
      n.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* s) { return dlsym(n.h, s); };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.send = reinterpret_cast<decltype(n.send)>(sym("ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(sym("ncclRecv"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    if (!n.get_unique_id || !n.comm_init_rank || !n.comm_destroy || !n.group_start ||
        !n.group_end || !n.send || !n.recv || !n.error_string) {
      n.err = "libnccl lacks ncclSend / ncclRecv / group entry points";
      n.h = nullptr;
    }
  });
  return n;
}

// ---------------------------------------------------------------- stream memory ops
struct MemOps {
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned) = nullptr;
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned) = nullptr;
};

const MemOps& memops() {
  static MemOps m;
  static std::once_flag once;
  std::call_once(once, [] {
    m.write32 = reinterpret_cast<decltype(m.write32)>(driver_entry("cuStreamWriteValue32"));
    m.wait32 = reinterpret_cast<decltype(m.wait32)>(driver_entry("cuStreamWaitValue32"));
  });
  return m;
}

constexpr int kFields = 3;  // exchanged fields: c, u_1, u_b (mask bits 1, 2, 4)
const char* const kFieldNames[kFields] = {"c", "u_1", "u_b"};
constexpr int kSets = 2;
// flag words per rank: [set][kind][side], kind 0 = "halo free" (written by the
// neighbour on `side`), 1 = "data arrived" (written by that neighbour)
constexpr int kFlagWords = kSets * 2 * 2;
inline int flag_index(int set, int kind, int side) { return (set * 2 + kind) * 2 + side; }
// connection probe words after the epoch flags: [side] written by a stream
// memory operation of the neighbour on `side`, [2 + side] by its copy engine
constexpr int kProbeWords = 4;
inline unsigned probe_token(int rank) { return 0x53500000u | (unsigned)(rank & 0xffff); }

// IPC blob: geometry + handles of every set's exchanged arrays + the flags
struct IpcEntry {
  cudaIpcMemHandle_t h;
  long long offset;
  int valid;
};
struct IpcBlob {
  int magic, rank, n, dtype, own0, own1, base, nplanes;
  IpcEntry arr[kSets][kFields];
  IpcEntry flags;
};
constexpr int kBlobMagic = 0x53474231;  // "SGB1"

}  // namespace
}  // namespace sgb

struct sgb_slab {
  std::string family;
  int n = 0, R = 0, rank = 0, world = 1, dtype = 4, transport = 0;
  int own0 = 0, own1 = 0, base = 0, nplanes = 0;
  std::vector<std::string> names;               // <family>_b array order
  void* arr[sgb::kSets][8] = {};                // bound device pointers
  cudaStream_t comm = nullptr;
  cudaEvent_t ev_done[sgb::kSets] = {}, ev_in = nullptr;
  unsigned epoch[sgb::kSets] = {0, 0};
  // NCCL
  ncclComm_t nccl = nullptr;
  // IPC
  unsigned* flags = nullptr;                    // kFlagWords + kProbeWords, this rank's memory
  unsigned* token = nullptr;                    // device word holding probe_token(rank)
  struct Peer {
    bool present = false, connected = false;
    int own0 = 0, own1 = 0, base = 0, nplanes = 0;
    void* arr[sgb::kSets][sgb::kFields] = {};   // neighbour's local arrays (mapped)
    unsigned* flags = nullptr;                  // neighbour's flag words (mapped)
    std::vector<std::pair<void*, long long>> opened;
  } peer[2];                                    // 0 = lower (rank-1), 1 = upper
};

namespace sgb {
namespace {

int fail(const std::string& msg) {
  set_error(msg);
  return SGB_EINVAL;
}
int cuda_fail(const char* what, cudaError_t e) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return -static_cast<int>(e);
}

int family_radius(const std::string& f) {
  if (f == "wave3d_r4") return 4;
  if (f == "wave3d_c" || f == "wave3d_c2") return 1;
  return 0;
}

int name_index(const sgb_slab* p, const char* name) {
  for (size_t i = 0; i < p->names.size(); i++)
    if (p->names[i] == name) return (int)i;
  return -1;
}

void* array_of(const sgb_slab* p, int set, const char* name) {
  const int i = name_index(p, name);
  if (i < 0) return nullptr;
  return p->arr[set][i] ? p->arr[set][i] : p->arr[0][i];
}

size_t plane_bytes(const sgb_slab* p) { return (size_t)p->n * p->n * p->dtype; }

// the exchange of `mask` fields of set `s` on the comm stream (after ev_in)
int exchange_nccl(sgb_slab* p, int s, unsigned mask) {
  Nccl& N = nccl();
  const size_t count = (size_t)p->R * p->n * p->n;
  const ncclDataType_t dt = p->dtype == 8 ? ncclFloat64 : ncclFloat32;
  const int lo = p->rank - 1, hi = p->rank + 1;
  ncclResult_t r = N.group_start();
  for (int f = 0; f < kFields && r == ncclSuccess; f++) {
    if (!(mask & (1u << f))) continue;
    char* a = static_cast<char*>(array_of(p, s, kFieldNames[f]));
    if (!a) return fail(std::string("sgb_slab: field '") + kFieldNames[f] + "' not bound");
    if (lo >= 0) {
      char* own_lo = a + (size_t)(p->own0 - p->base) * plane_bytes(p);
      if (r == ncclSuccess) r = N.send(own_lo, count, dt, lo, p->nccl, p->comm);
      if (r == ncclSuccess) r = N.recv(a, count, dt, lo, p->nccl, p->comm);
    }
    if (hi < p->world) {
      char* own_hi = a + (size_t)(p->own1 - p->R - p->base) * plane_bytes(p);
      char* halo_hi = a + (size_t)(p->own1 - p->base) * plane_bytes(p);
      if (r == ncclSuccess) r = N.send(own_hi, count, dt, hi, p->nccl, p->comm);
      if (r == ncclSuccess) r = N.recv(halo_hi, count, dt, hi, p->nccl, p->comm);
    }
  }
  const ncclResult_t r2 = N.group_end();
  if (r == ncclSuccess) r = r2;
  if (r != ncclSuccess) return fail(std::string("NCCL halo exchange: ") + N.error_string(r));
  return 0;
}

int exchange_ipc(sgb_slab* p, int s, unsigned mask, unsigned e) {
  const MemOps& M = memops();
  if (!M.write32 || !M.wait32) return fail("stream memory operations unavailable");
  CUstream cs = reinterpret_cast<CUstream>(p->comm);
  // 1. tell each neighbour our halo of set s is free for epoch e (every prior
  //    reader of it is ordered before ev_in)
  for (int side = 0; side < 2; side++) {
    const auto& nb = p->peer[side];
    if (!nb.present) continue;
    // we are the neighbour's side (1 - side)
    CUdeviceptr w = (CUdeviceptr)(nb.flags + flag_index(s, 0, 1 - side));
    if (M.write32(cs, w, e, 0) != CUDA_SUCCESS) return fail("cuStreamWriteValue32 (ready)");
  }
  // 2. per neighbour: wait until its halo is free, push our edge planes, and
  //    tell it the data of epoch e arrived
  const size_t bytes = (size_t)p->R * plane_bytes(p);
  for (int side = 0; side < 2; side++) {
    const auto& nb = p->peer[side];
    if (!nb.present) continue;
    CUdeviceptr mine = (CUdeviceptr)(p->flags + flag_index(s, 0, side));
    if (M.wait32(cs, mine, e, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return fail("cuStreamWaitValue32 (ready)");
    for (int f = 0; f < kFields; f++) {
      if (!(mask & (1u << f))) continue;
      const char* a = static_cast<const char*>(array_of(p, s, kFieldNames[f]));
      char* d = static_cast<char*>(nb.arr[s][f] ? nb.arr[s][f] : nb.arr[0][f]);
      if (!a || !d) return fail(std::string("sgb_slab: field '") + kFieldNames[f] + "' not bound");
      // lower neighbour's upper halo = global planes [own0, own0 + R); upper
      // neighbour's lower halo = [own1 - R, own1)
      const int g0 = side == 0 ? p->own0 : p->own1 - p->R;
      const char* src = a + (size_t)(g0 - p->base) * plane_bytes(p);
      char* dst = d + (size_t)(g0 - nb.base) * plane_bytes(p);
      const cudaError_t ce = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, p->comm);
      if (ce != cudaSuccess) return cuda_fail("halo push", ce);
    }
    CUdeviceptr w = (CUdeviceptr)(nb.flags + flag_index(s, 1, 1 - side));
    if (M.write32(cs, w, e, 0) != CUDA_SUCCESS) return fail("cuStreamWriteValue32 (arrived)");
  }
  return 0;
}

int wait_ipc_arrival(sgb_slab* p, int s, cudaStream_t st) {
  const MemOps& M = memops();
  for (int side = 0; side < 2; side++) {
    if (!p->peer[side].present) continue;
    CUdeviceptr mine = (CUdeviceptr)(p->flags + flag_index(s, 1, side));
    if (M.wait32(reinterpret_cast<CUstream>(st), mine, p->epoch[s], CU_STREAM_WAIT_VALUE_GEQ) !=
        CUDA_SUCCESS)
      return fail("cuStreamWaitValue32 (arrived)");
  }
  return 0;
}

int gather(sgb_slab* p, int s, const double* sc, bool fresh, int o0, int o1, cudaStream_t st) {
  if (o1 <= o0) return 0;
  void* c = array_of(p, s, "c");
  void* cb = array_of(p, s, "c_b");
  void* u1 = array_of(p, s, "u_1");
  void* u1b = array_of(p, s, "u_1_b");
  void* ub = array_of(p, s, "u_b");
  void* u2b = array_of(p, s, "u_2_b");
  if (!c || !cb || !u1 || !u1b || !ub || (p->R == 1 && !u2b))
    return fail("sgb_slab_step: arrays not bound");
  sgb_stream_t ss = reinterpret_cast<sgb_stream_t>(st);
  const int n = p->n, b = p->base, np = p->nplanes;
  if (p->family == "wave3d_r4") {
    if (p->dtype == 4) {
      if (fresh)
        return wave3d_r4_b_fresh_slab_f32(n, sc[0], (float*)c, (float*)cb, (float*)u1,
                                          (float*)u1b, (float*)ub, b, np, o0, o1, ss);
      return wave3d_r4_b_slab_f32(n, sc[0], (float*)c, (float*)cb, (float*)u1, (float*)u1b,
                                  (float*)ub, b, np, o0, o1, ss);
    }
    if (fresh)
      return wave3d_r4_b_fresh_slab_f64(n, sc[0], (double*)c, (double*)cb, (double*)u1,
                                        (double*)u1b, (double*)ub, b, np, o0, o1, ss);
    return wave3d_r4_b_slab_f64(n, sc[0], (double*)c, (double*)cb, (double*)u1, (double*)u1b,
                                (double*)ub, b, np, o0, o1, ss);
  }
  if (fresh) return fail("sgb_slab_step: SGB_STEP_FRESH is a wave3d_r4 form");
  if (p->family != "wave3d_c") return fail("sgb_slab_step: unsupported family " + p->family);
  if (p->dtype == 4)
    return wave3d_c_b_slab_f32(n, sc[0], (float*)c, (float*)cb, (float*)u1, (float*)u1b,
                               (float*)u2b, (float*)ub, b, np, o0, o1, ss);
  return wave3d_c_b_slab_f64(n, sc[0], (double*)c, (double*)cb, (double*)u1, (double*)u1b,
                             (double*)u2b, (double*)ub, b, np, o0, o1, ss);
}

}  // namespace
}  // namespace sgb

using namespace sgb;

extern "C" {

int sgb_slab_decompose(int n, int radius, int world, int rank, int* own0, int* own1, int* base,
                       int* nplanes) {
  if (world < 1 || rank < 0 || rank >= world || radius < 0 || n < world * radius || n <= 0)
    return fail("sgb_slab_decompose: bad n / radius / world / rank");
  const int q = n / world, r = n % world;
  const int o0 = rank * q + (rank < r ? rank : r);
  const int o1 = o0 + q + (rank < r ? 1 : 0);
  const int lo = rank > 0 ? radius : 0, hi = rank < world - 1 ? radius : 0;
  if (own0) *own0 = o0;
  if (own1) *own1 = o1;
  if (base) *base = o0 - lo;
  if (nplanes) *nplanes = o1 - o0 + lo + hi;
  return 0;
}

int sgb_nccl_unique_id(void* id128) {
  Nccl& N = nccl();
  if (!N.h) return fail(N.err);
  ncclUniqueId id;
  const ncclResult_t r = N.get_unique_id(&id);
  if (r != ncclSuccess) return fail(std::string("ncclGetUniqueId: ") + N.error_string(r));
  std::memcpy(id128, &id, sizeof(id));
  return 0;
}

sgb_slab* sgb_slab_create(const char* family, int n, int dtype_bytes, int rank, int world,
                          int transport, const void* nccl_id128) {
  const std::string fam = family ? family : "";
  const int R = family_radius(fam);
  if (!R || (fam == "wave3d_c2")) {
    set_error("sgb_slab_create: z-slab plans exist for wave3d_r4 and wave3d_c");
    return nullptr;
  }
  if (dtype_bytes != 4 && dtype_bytes != 8) {
    set_error("sgb_slab_create: dtype_bytes must be 4 or 8");
    return nullptr;
  }
  if (transport != SGB_TRANSPORT_NCCL && transport != SGB_TRANSPORT_IPC) {
    set_error("sgb_slab_create: unknown transport");
    return nullptr;
  }
  auto* p = new sgb_slab;
  p->family = fam;
  p->n = n;
  p->R = R;
  p->rank = rank;
  p->world = world;
  p->dtype = dtype_bytes;
  p->transport = transport;
  if (sgb_slab_decompose(n, R, world, rank, &p->own0, &p->own1, &p->base, &p->nplanes) != 0) {
    delete p;
    return nullptr;
  }
  p->names = R == 4 ? std::vector<std::string>{"c", "c_b", "u_1", "u_1_b", "u_b"}
                    : std::vector<std::string>{"c", "c_b", "u_1", "u_1_b", "u_2_b", "u_b"};
  cudaError_t e = cudaStreamCreateWithPriority(&p->comm, cudaStreamNonBlocking, -1);
  for (int s = 0; s < kSets && e == cudaSuccess; s++) {
    e = cudaEventCreateWithFlags(&p->ev_done[s], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    cuda_fail("sgb_slab_create", e);
    sgb_slab_destroy(p);
    return nullptr;
  }
  if (transport == SGB_TRANSPORT_NCCL && world > 1) {
    Nccl& N = nccl();
    if (!N.h || !nccl_id128) {
      set_error(N.h ? "sgb_slab_create: NCCL transport needs the unique id" : N.err);
      sgb_slab_destroy(p);
      return nullptr;
    }
    ncclUniqueId id;
    std::memcpy(&id, nccl_id128, sizeof(id));
    const ncclResult_t r = N.comm_init_rank(&p->nccl, world, id, rank);
    if (r != ncclSuccess) {
      set_error(std::string("ncclCommInitRank: ") + N.error_string(r));
      p->nccl = nullptr;
      sgb_slab_destroy(p);
      return nullptr;
    }
  }
  if (transport == SGB_TRANSPORT_IPC) {
    e = cudaMalloc(&p->flags, (kFlagWords + kProbeWords) * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(p->flags, 0, (kFlagWords + kProbeWords) * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      cuda_fail("sgb_slab_create (flags)", e);
      sgb_slab_destroy(p);
      return nullptr;
    }
    p->peer[0].present = rank > 0;
    p->peer[1].present = rank < world - 1;
  }
  return p;
}

int sgb_slab_geometry(const sgb_slab* p, int* base, int* nplanes, int* own0, int* own1) {
  if (!p) return fail("sgb_slab_geometry: null plan");
  if (base) *base = p->base;
  if (nplanes) *nplanes = p->nplanes;
  if (own0) *own0 = p->own0;
  if (own1) *own1 = p->own1;
  return 0;
}

int sgb_slab_bind(sgb_slab* p, int set, const char* name, void* device_ptr) {
  if (!p || set < 0 || set >= kSets || !name) return fail("sgb_slab_bind: bad arguments");
  const int i = name_index(p, name);
  if (i < 0) return fail(std::string("sgb_slab_bind: '") + name + "' is not an array of " +
                         p->family + "_b");
  if (device_ptr && (reinterpret_cast<uintptr_t>(device_ptr) & 15))
    return fail("sgb_slab_bind: arrays must be 16-byte aligned");
  if (p->transport == SGB_TRANSPORT_IPC && (p->peer[0].connected || p->peer[1].connected)) {
    for (int f = 0; f < kFields; f++)
      if (std::strcmp(name, kFieldNames[f]) == 0)
        return fail("sgb_slab_bind: exchanged fields are fixed once IPC is connected");
  }
  p->arr[set][i] = device_ptr;
  return 0;
}

int sgb_slab_ipc_export(const sgb_slab* p, void* blob, long long* bytes) {
  if (!p || p->transport != SGB_TRANSPORT_IPC) return fail("sgb_slab_ipc_export: not an IPC plan");
  if (bytes) {
    const long long cap = *bytes;
    *bytes = (long long)sizeof(IpcBlob);
    if (!blob) return 0;
    if (cap < (long long)sizeof(IpcBlob)) return fail("sgb_slab_ipc_export: blob too small");
  }
  if (!blob) return fail("sgb_slab_ipc_export: null blob");
  IpcBlob b;
  std::memset(&b, 0, sizeof(b));
  b.magic = kBlobMagic;
  b.rank = p->rank;
  b.n = p->n;
  b.dtype = p->dtype;
  b.own0 = p->own0;
  b.own1 = p->own1;
  b.base = p->base;
  b.nplanes = p->nplanes;
  for (int s = 0; s < kSets; s++)
    for (int f = 0; f < kFields; f++) {
      const int i = name_index(p, kFieldNames[f]);
      void* a = p->arr[s][i];
      if (!a) continue;
      if (int rc = sgb_ipc_handle(a, &b.arr[s][f].h, &b.arr[s][f].offset)) return rc;
      b.arr[s][f].valid = 1;
    }
  if (int rc = sgb_ipc_handle(p->flags, &b.flags.h, &b.flags.offset)) return rc;
  b.flags.valid = 1;
  std::memcpy(blob, &b, sizeof(b));
  return 0;
}

int sgb_slab_ipc_connect(sgb_slab* p, const void* lower_blob, const void* upper_blob) {
  if (!p || p->transport != SGB_TRANSPORT_IPC) return fail("sgb_slab_ipc_connect: not an IPC plan");
  const void* blobs[2] = {lower_blob, upper_blob};
  for (int side = 0; side < 2; side++) {
    auto& nb = p->peer[side];
    if (!nb.present) continue;
    if (!blobs[side]) return fail("sgb_slab_ipc_connect: missing neighbour blob");
    IpcBlob b;
    std::memcpy(&b, blobs[side], sizeof(b));
    const int want_rank = p->rank + (side == 0 ? -1 : 1);
    if (b.magic != kBlobMagic || b.rank != want_rank || b.n != p->n || b.dtype != p->dtype)
      return fail("sgb_slab_ipc_connect: neighbour blob does not match this plan");
    // the planes pushed into the neighbour's halo must lie in its local array
    const int g0 = side == 0 ? p->own0 : p->own1 - p->R;
    if (g0 < b.base || g0 + p->R > b.base + b.nplanes)
      return fail("sgb_slab_ipc_connect: neighbour halo planes do not line up");
    nb.own0 = b.own0;
    nb.own1 = b.own1;
    nb.base = b.base;
    nb.nplanes = b.nplanes;
    for (int s = 0; s < kSets; s++)
      for (int f = 0; f < kFields; f++) {
        if (!b.arr[s][f].valid) continue;
        void* ptr = nullptr;
        if (int rc = sgb_ipc_open(&b.arr[s][f].h, b.arr[s][f].offset, &ptr)) return rc;
        nb.arr[s][f] = ptr;
        nb.opened.emplace_back(ptr, b.arr[s][f].offset);
      }
    void* fl = nullptr;
    if (int rc = sgb_ipc_open(&b.flags.h, b.flags.offset, &fl)) return rc;
    nb.flags = static_cast<unsigned*>(fl);
    nb.opened.emplace_back(fl, b.flags.offset);
    nb.connected = true;
  }
  return 0;
}

int sgb_slab_ipc_probe(sgb_slab* p, int phase) {
  if (!p || p->transport != SGB_TRANSPORT_IPC) return fail("sgb_slab_ipc_probe: not an IPC plan");
  if (phase == 0) {
    // write our token into each neighbour's probe words: once by a stream
    // memory operation (the epoch flags' path), once by a copy-engine copy
    // (the halo planes' path); neither can block
    const MemOps& M = memops();
    if (!M.write32) return fail("stream memory operations unavailable");
    if (!p->token) {
      cudaError_t e = cudaMalloc(&p->token, sizeof(unsigned));
      const unsigned t = probe_token(p->rank);
      if (e == cudaSuccess) e = cudaMemcpy(p->token, &t, sizeof(t), cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_fail("sgb_slab_ipc_probe", e);
    }
    CUstream cs = reinterpret_cast<CUstream>(p->comm);
    for (int side = 0; side < 2; side++) {
      const auto& nb = p->peer[side];
      if (!nb.present) continue;
      if (!nb.connected) return fail("sgb_slab_ipc_probe: neighbours not connected");
      unsigned* w = nb.flags + kFlagWords;
      if (M.write32(cs, (CUdeviceptr)(w + (1 - side)), probe_token(p->rank), 0) != CUDA_SUCCESS)
        return fail("sgb_slab_ipc_probe: remote cuStreamWriteValue32 failed");
      const cudaError_t e = cudaMemcpyAsync(w + 2 + (1 - side), p->token, sizeof(unsigned),
                                            cudaMemcpyDeviceToDevice, p->comm);
      if (e != cudaSuccess) return cuda_fail("sgb_slab_ipc_probe (peer copy)", e);
    }
    const cudaError_t e = cudaStreamSynchronize(p->comm);
    return e == cudaSuccess ? 0 : cuda_fail("sgb_slab_ipc_probe", e);
  }
  // phase 1 (after every rank's phase 0): both tokens of each neighbour arrived
  unsigned w[kProbeWords];
  const cudaError_t e =
      cudaMemcpy(w, p->flags + kFlagWords, sizeof(w), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_fail("sgb_slab_ipc_probe", e);
  for (int side = 0; side < 2; side++) {
    if (!p->peer[side].present) continue;
    const unsigned want = probe_token(p->rank + (side == 0 ? -1 : 1));
    if (w[side] != want || w[2 + side] != want)
      return fail("sgb_slab_ipc_probe: the " + std::string(side == 0 ? "lower" : "upper") +
                  " neighbour's remote writes did not arrive (no usable peer path)");
  }
  return 0;
}

int sgb_slab_release(sgb_slab* p) {
  if (!p || p->transport != SGB_TRANSPORT_IPC) return fail("sgb_slab_release: not an IPC plan");
  // watchdog's last resort: satisfy every wait on this rank's flags (cyclic
  // GEQ compare) from a fresh stream, so a stuck exchange drains; the plan's
  // results are void afterwards and it must be destroyed
  unsigned v[kFlagWords];
  for (int s = 0; s < kSets; s++)
    for (int i = 0; i < 4; i++) v[s * 4 + i] = p->epoch[s] + (1u << 30);
  cudaStream_t st = nullptr;
  cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMemcpyAsync(p->flags, v, sizeof(v), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (st) cudaStreamDestroy(st);
  return e == cudaSuccess ? 0 : cuda_fail("sgb_slab_release", e);
}

int sgb_slab_halo_start(sgb_slab* p, int set, unsigned fields_mask, sgb_stream_t stream) {
  if (!p || set < 0 || set >= kSets) return fail("sgb_slab_halo_start: bad arguments");
  cudaStream_t st = as_stream(stream);
  p->epoch[set]++;
  if (p->world == 1 || !fields_mask) {
    const cudaError_t e = cudaEventRecord(p->ev_done[set], st);
    return e == cudaSuccess ? 0 : cuda_fail("sgb_slab_halo_start", e);
  }
  if (p->transport == SGB_TRANSPORT_IPC &&
      ((p->peer[0].present && !p->peer[0].connected) ||
       (p->peer[1].present && !p->peer[1].connected)))
    return fail("sgb_slab_halo_start: IPC neighbours not connected (sgb_slab_ipc_connect)");
  cudaError_t e = cudaEventRecord(p->ev_in, st);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->comm, p->ev_in, 0);
  if (e != cudaSuccess) return cuda_fail("sgb_slab_halo_start", e);
  const int rc = p->transport == SGB_TRANSPORT_NCCL ? exchange_nccl(p, set, fields_mask)
                                                    : exchange_ipc(p, set, fields_mask,
                                                                   p->epoch[set]);
  if (rc) return rc;
  e = cudaEventRecord(p->ev_done[set], p->comm);
  return e == cudaSuccess ? 0 : cuda_fail("sgb_slab_halo_start", e);
}

int sgb_slab_halo_wait(sgb_slab* p, int set, sgb_stream_t stream) {
  if (!p || set < 0 || set >= kSets) return fail("sgb_slab_halo_wait: bad arguments");
  cudaStream_t st = as_stream(stream);
  // our own pushes / sends are done (the source planes may be overwritten)...
  const cudaError_t e = cudaStreamWaitEvent(st, p->ev_done[set], 0);
  if (e != cudaSuccess) return cuda_fail("sgb_slab_halo_wait", e);
  // ... and (IPC) the neighbours' pushes into our halos arrived
  if (p->transport == SGB_TRANSPORT_IPC && p->world > 1) return wait_ipc_arrival(p, set, st);
  return 0;
}

int sgb_slab_step(sgb_slab* p, int set, const double* scalars, int flags, sgb_stream_t stream) {
  if (!p || !scalars || set < 0 || set >= kSets) return fail("sgb_slab_step: bad arguments");
  cudaStream_t st = as_stream(stream);
  const bool fresh = flags & SGB_STEP_FRESH;
  const unsigned mask = 2u | 4u;  // u_1, u_b
  if (flags & SGB_STEP_NO_EXCHANGE) {  // halos of `set` exchanged earlier (pipelined)
    if (int rc = sgb_slab_halo_wait(p, set, stream)) return rc;
    return gather(p, set, scalars, fresh, p->own0, p->own1, st);
  }
  if (int rc = sgb_slab_halo_start(p, set, mask, stream)) return rc;
  const int R = p->R;
  const int lo_in = p->own0 + (p->rank > 0 ? R : 0);
  const int hi_in = p->own1 - (p->rank < p->world - 1 ? R : 0);
  if (!(flags & SGB_STEP_OVERLAP) || hi_in <= lo_in || p->world == 1) {
    if (int rc = sgb_slab_halo_wait(p, set, stream)) return rc;
    return gather(p, set, scalars, fresh, p->own0, p->own1, st);
  }
  // interior planes (their stencils read only owned planes) during the
  // exchange, then the two edge bands
  if (int rc = gather(p, set, scalars, fresh, lo_in, hi_in, st)) return rc;
  if (int rc = sgb_slab_halo_wait(p, set, stream)) return rc;
  if (int rc = gather(p, set, scalars, fresh, p->own0, lo_in, st)) return rc;
  return gather(p, set, scalars, fresh, hi_in, p->own1, st);
}

void sgb_slab_destroy(sgb_slab* p) {
  if (!p) return;
  if (p->comm) cudaStreamSynchronize(p->comm);
  if (p->nccl) nccl().comm_destroy(p->nccl);
  for (auto& nb : p->peer)
    for (auto& o : nb.opened) sgb_ipc_close(o.first, o.second);
  if (p->flags) cudaFree(p->flags);
  if (p->token) cudaFree(p->token);
  for (int s = 0; s < kSets; s++) {
    if (p->ev_done[s]) cudaEventDestroy(p->ev_done[s]);
  }
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->comm) cudaStreamDestroy(p->comm);
  delete p;
}

}  // extern "C"
