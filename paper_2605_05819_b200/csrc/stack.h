// Persistent decode-stack kernel: one cooperative launch runs every compensation window of
// hc_stack_forward (QKV -> O -> UPGATE -> DOWN per layer) with the weight stream never
// stopping at a window boundary (opt-in HC_STACK_KERNEL=1).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "decode.h"

namespace hc {

// One window of the plan (device table entry): the per-window decode arguments (members, x' input,
// y / y16 outputs, residual, glue, t accumulators, t forwarding) and the CTA rotation.
struct SWin {
  DArgs a;
  int rot;        // item i of this window runs on CTA (i + rot) % grid (balances CTAs across windows)
  int pad;
};

struct StackArgs {
  const SWin* wins;   // [n_win], device
  int n_win;
  int n_vwarps0;      // V warps of window 0 (its t is computed in-kernel; later windows' t is forwarded)
  unsigned* done;     // [n_win] row blocks completed per window (zeroed before every launch)
  unsigned* vdone;    // [1] window-0 V warps completed (zeroed before every launch)
};

size_t stack_smem_bytes();
// V warps of window 0 with n_vp rank-projection pieces on a grid of `grid` CTAs (host + device rule).
int stack_vwarps(int n_vp, int grid);
// Co-resident CTAs of the stack kernel (its grid), 0 if it cannot run.
int stack_grid(int bits, size_t smem);
cudaError_t launch_stack(const StackArgs& s, int bits, int grid, size_t smem, cudaStream_t st);

}  // namespace hc
