// NCCL is loaded with dlopen("libnccl.so.2") so the library has no link-time NCCL dependency and
// shares the copy the process (e.g. PyTorch) already loaded.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>

#include "comm.h"
#include "hcinfer.h"

namespace hc {

namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

NcclApi* api(char* msg, int len) {
  static NcclApi a;
  static bool tried = false;
  if (!tried) {
    tried = true;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) a.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (a.h) {
      a.getUniqueId = (decltype(a.getUniqueId))dlsym(a.h, "ncclGetUniqueId");
      a.commInitRank = (decltype(a.commInitRank))dlsym(a.h, "ncclCommInitRank");
      a.commDestroy = (decltype(a.commDestroy))dlsym(a.h, "ncclCommDestroy");
      a.allGather = (decltype(a.allGather))dlsym(a.h, "ncclAllGather");
      a.errStr = (decltype(a.errStr))dlsym(a.h, "ncclGetErrorString");
    }
  }
  if (!a.h || !a.getUniqueId || !a.commInitRank || !a.commDestroy || !a.allGather || !a.errStr) {
    snprintf(msg, len, "NCCL not available (dlopen libnccl.so.2: %s)", dlerror() ? dlerror() : "symbols missing");
    return nullptr;
  }
  return &a;
}
}  // namespace

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
};

bool comm_unique_id(uint8_t* out128, char* msg, int len) {
  NcclApi* a = api(msg, len);
  if (!a) return false;
  ncclUniqueId id;
  ncclResult_t r = a->getUniqueId(&id);
  if (r != ncclSuccess) { snprintf(msg, len, "ncclGetUniqueId: %s", a->errStr(r)); return false; }
  for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) out128[i] = (uint8_t)id.internal[i];
  return true;
}

Comm* comm_create(const uint8_t* id128, int rank, int world, char* msg, int len) {
  NcclApi* a = api(msg, len);
  if (!a) return nullptr;
  ncclUniqueId id;
  for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) id.internal[i] = (char)id128[i];
  Comm* c = new Comm();
  ncclResult_t r = a->commInitRank(&c->comm, world, id, rank);
  if (r != ncclSuccess) {
    snprintf(msg, len, "ncclCommInitRank(rank %d of %d): %s", rank, world, a->errStr(r));
    delete c;
    return nullptr;
  }
  c->rank = rank;
  c->world = world;
  return c;
}

void comm_destroy(Comm* c) {
  if (!c) return;
  char m[8];
  NcclApi* a = api(m, 8);
  if (a && c->comm) a->commDestroy(c->comm);
  delete c;
}

bool comm_allgather_bf16(Comm* c, const void* send, void* recv, size_t count, cudaStream_t st, char* msg, int len) {
  NcclApi* a = api(msg, len);
  if (!a) return false;
  ncclResult_t r = a->allGather(send, recv, count, ncclBfloat16, c->comm, st);
  if (r != ncclSuccess) { snprintf(msg, len, "ncclAllGather: %s", a->errStr(r)); return false; }
  return true;
}

// one thread per (b, full column)
__global__ void unshard_kernel(const uint16_t* __restrict__ g, uint16_t* __restrict__ out, GatherPlan gp) {
  const int n_full = gp.G * gp.n_local;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)gp.B * n_full) return;
  const int b = (int)(i / n_full), col = (int)(i % n_full);
  out[i] = g[unshard_src(gp, b, col)];
}

cudaError_t launch_unshard(const uint16_t* gathered, uint16_t* out, const GatherPlan& gp, cudaStream_t st) {
  const long long n = (long long)gp.B * gp.G * gp.n_local;
  unshard_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(gathered, out, gp);
  return cudaGetLastError();
}

}  // namespace hc

extern "C" hc_status hc_unshard_host(const uint16_t* gathered, uint16_t* out, int32_t G, int32_t B, int32_t n_members,
                               const int32_t* widths) {
  if (!gathered || !out || !widths || G < 1 || B < 1 || n_members < 1 || n_members > 4) return HC_ERR_CONFIG;
  hc::GatherPlan gp{};
  gp.G = G; gp.B = B; gp.n_members = n_members;
  int o = 0;
  for (int i = 0; i < n_members; ++i) { gp.w[i] = widths[i]; gp.o[i] = o; o += widths[i]; }
  gp.n_local = o;
  for (int b = 0; b < B; ++b)
    for (int col = 0; col < G * o; ++col) out[(size_t)b * G * o + col] = gathered[hc::unshard_src(gp, b, col)];
  return HC_OK;
}
