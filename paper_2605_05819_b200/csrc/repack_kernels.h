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
// fp8 (e4m3) factors: U8 fragments [rb][c][lane][8 B] of n_rb row blocks (rows from U0 / U1
// as RepackSrc) and V8 pieces [c][g][j][lane][8 B]; *nan_flag |= 1 on a NaN encoding.
cudaError_t launch_repack_fp8(const uint8_t* U0, const uint8_t* U1, int rstride, int n_rb, const uint8_t* V, int K,
                              int r_stored, uint8_t* u_out, uint8_t* v_out, unsigned* nan_flag, cudaStream_t st);
// fp16(e4m3 · per-rank scale) copies for the prefill path; rank_major: [r_stored][K] (V), else [rows][r_stored] (U).
cudaError_t launch_fp8_to_f16(const uint8_t* in, const float* scale, size_t n, int r_stored, bool rank_major, int K,
                              uint16_t* out, cudaStream_t st);
// Lazy prefill copies (4-bit plain members): decode records -> canonical 4-bit codes [rows][K/8] (via q bytes
// [rows][K] in q_tmp), scales / zeros [rows][G]; U / V fragments (bf16, or fp8 with scales us / vs) -> fp16
// U [rows][r_stored] and V [r_stored][K].
cudaError_t launch_unrepack_prefill(const uint8_t* rec, int n_rb, int K, int bits, uint8_t* q_tmp, uint32_t* codes_out,
                                    uint16_t* scales_out, uint8_t* zeros_out, const uint8_t* Ufrag, const uint8_t* Vfrag,
                                    int r_stored, const float* us, const float* vs, uint16_t* U16, uint16_t* V16,
                                    cudaStream_t st);
}  // namespace hc
