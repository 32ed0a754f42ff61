// Process-wide development switches (hc_set_option / hc_get_option in include/hcinfer.h).  They select
// between measured-equivalent plans for A/B timing; every setting computes the same product within the
// fp32 rounding of its accumulation order (all parity tests pass under each).  Read when a window plan or a
// stack graph is built; a change bumps `epoch` so that contexts re-capture their graphs.
#pragma once

namespace hc {

struct Options {
  int t_forward = 0;           // stack: the producer window accumulates the next window's t = V·x
  int x_handoff = 1;           // stack: producer epilogue writes the next fp16-path window's x' (§7.1)
  int dep_wait = 1;            // stack: dataflow dependency on the producer's counter instead of the grid boundary
  int int8_path = 1;           // decode: u8·s8 tensor-core path for 2/4-bit at B <= 2 (decode_i8.cuh)
  int prefill_merge = 1;       // prefill: one GEMM over a multi-member window
  int decode_ctas_per_sm = 0;  // decode: cap on resident CTAs per SM (0 = occupancy limit)
  int pdl = 1;                 // decode: programmatic dependent launch between windows
  int l2_prefetch = 0;         // stack: next-window record items each CTA prefetches into L2 (0 = off)
  int l2_prefetch_at_start = 0;   // stack: issue them at kernel start (spare producer lanes) instead of after the ring
  unsigned epoch = 0;
};

Options& options();

}  // namespace hc
