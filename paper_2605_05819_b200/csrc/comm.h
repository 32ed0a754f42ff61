// Multi-GPU column sharding support: NCCL (loaded at run time) and the gather permute.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hc {

struct Comm;   // opaque: dlopen'ed NCCL + communicator

// NCCL unique id (128 bytes) for rank 0 to broadcast.  Returns false (msg set) on failure.
bool comm_unique_id(uint8_t* out128, char* msg, int msg_len);
// ncclCommInitRank on the current device.  nullptr (msg set) on failure.
Comm* comm_create(const uint8_t* id128, int rank, int world, char* msg, int msg_len);
void comm_destroy(Comm* c);
// ncclAllGather of `count` bf16 elements per rank on `st` (recv = [world][count]).
bool comm_allgather_bf16(Comm* c, const void* send, void* recv, size_t count, cudaStream_t st, char* msg, int msg_len);

// Gathered slices [G][B][n_local] -> canonical [B][N_full] for a window of n_members members, member m
// having w[m] local rows at local offset o[m] (full offset F[m] = Σ_{m'<m} G·w[m']).
struct GatherPlan {
  int G, B, n_local, n_members;
  int w[4], o[4];
};
cudaError_t launch_unshard(const uint16_t* gathered, uint16_t* out, const GatherPlan& gp, cudaStream_t st);

// Source index in the gathered buffer of output element (b, col): shared by the kernel and the host
// test export hc_unshard_host.
#ifdef __CUDACC__
__host__ __device__
#endif
inline size_t unshard_src(const GatherPlan& gp, int b, int col) {
  int base = 0, m = 0;
  for (; m < gp.n_members - 1; ++m) {
    if (col < base + gp.G * gp.w[m]) break;
    base += gp.G * gp.w[m];
  }
  const int j = col - base, p = j / gp.w[m], jj = j % gp.w[m];
  return ((size_t)p * gp.B + b) * gp.n_local + gp.o[m] + jj;
}

}  // namespace hc
