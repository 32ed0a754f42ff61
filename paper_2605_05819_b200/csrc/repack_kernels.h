#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hc {
// Row sources of a repack: row r of row block rb is taken from [0] (r < 8) or [1] (r >= 8),
// source row rb*rstride + (r & 7) (repack.cuh row_ptr).
struct RepackSrc {
  const uint32_t* codes[2];
  const uint16_t* scales[2];
  const uint8_t* zeros[2];
  const uint16_t* U[2];
  int rstride;
};
// Kernel records (codes+scales+zeros) and U fragments of n_rb row blocks (layout.h).
cudaError_t launch_repack_records(const RepackSrc& src, int K, int bits, int r_stored, int n_rb, uint8_t* rec_out,
                                  uint32_t* u_out, cudaStream_t st);
// V fragments [c][g][j][lane][4] of one matrix.
cudaError_t launch_repack_v(const uint16_t* V, int K, int r_stored, uint32_t* v_out, cudaStream_t st);
// Natural-k V fragments [K/16][c][lane][4] (standard m16n8k16 A layout: ranks = rows, 16 consecutive k)
// for t forwarding (DArgs::fwd_vn).
cudaError_t launch_repack_vn(const uint16_t* V, int K, int r_stored, uint32_t* out, cudaStream_t st);
}  // namespace hc
