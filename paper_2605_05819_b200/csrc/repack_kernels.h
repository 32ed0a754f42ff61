#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hc {
// Repack rows [row0, row0 + n_rows) of one matrix (device pointers) into kernel records,
// U tiles and V tiles (layout.h).  u_out / v_out unused when r_stored == 0.
cudaError_t launch_repack(const uint32_t* codes, const uint16_t* scales, const uint8_t* zeros,
                          const uint16_t* U, const uint16_t* V, int K, int bits, int r_stored,
                          int row0, int n_rows, uint8_t* rec_out, uint32_t* u_out, uint32_t* v_out,
                          cudaStream_t st);
}  // namespace hc
