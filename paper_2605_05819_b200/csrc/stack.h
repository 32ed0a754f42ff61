// Persistent decode-stack kernel: one launch runs every compensation window of hc_stack_forward
// (QKV -> O -> UPGATE -> DOWN per layer) with the weight stream never stopping at a
// window boundary.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "decode.h"

#ifndef HC_STK_TPB
#define HC_STK_TPB 2
#endif
#ifndef HC_STK_NBUF
#define HC_STK_NBUF 3
#endif
#ifndef HC_STK_RED
#define HC_STK_RED 4
#endif

namespace hc {

constexpr int kSW = 16;                      // tile warps per CTA (one CTA per SM)
constexpr int kSThreads = (kSW + 1) * 32;    // + the epilogue warp
constexpr int kSTPB = HC_STK_TPB;            // tiles per bulk-copy block
constexpr int kSNBuf = HC_STK_NBUF;          // blocks per tile-warp ring
constexpr int kSRed = HC_STK_RED;            // partial-sum hand-off slots (items in flight per CTA)

// One window of the plan (device table entry).  `a` is the per-window argument block of the
// decode kernel (members, x / y / residual pointers, glue, rank chunks, t accumulators); a.cnt
// is unused here (the stack kernel keeps its counters in StackArgs).
struct SWin {
  DArgs a;
  int rot;        // item i of this window runs on CTA (i + rot) % grid (balances CTAs across windows)
  int n_vwarps;   // tile warps that hold rank-projection (V·x) pieces of this window
};

struct StackArgs {
  const SWin* wins;   // [n_win], device
  int n_win;
  int xs_ld;          // shared x' row stride (elements) = max K + 32
  int u_slot_chunks;  // U prefetch slot size in 16-rank chunks (max over the plan's windows)
  int n_uslots;       // U prefetch slots (2..8): U of n_uslots - 1 items ahead of the epilogue
  unsigned* done;     // [n_win] row blocks completed per window (zeroed before every launch)
  unsigned* vdone;    // [n_win] V warps completed per window (zeroed before every launch)
};

// Shared memory of the stack kernel for batch B, the largest K of the plan and its U prefetch ring;
// 0 if it cannot fit.
size_t stack_smem_bytes(int B, int k_max, int u_slot_chunks, int n_uslots);
int stack_uslots_max();
// V warps of a window with n_vp rank-projection pieces on a grid of `grid` CTAs (host + device rule).
int stack_vwarps(int n_vp, int grid);
// Co-resident CTAs of the stack kernel (its grid), 0 if it cannot run.
int stack_grid(int bits, size_t smem);
cudaError_t stack_set_trace(void* buf);
cudaError_t stack_set_acct(void* buf);     // dev: per-warp cycle accounting [grid][17][4] (HC_STK_TRACE builds)   // dev: globaltimer trace buffer [n_win][grid][4] (HC_STK_TRACE builds)
cudaError_t launch_stack(const StackArgs& s, int bits, int grid, size_t smem, cudaStream_t st);

}  // namespace hc
