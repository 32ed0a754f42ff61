// Prefill / batched path: tcgen05 (5th-gen tensor core) compensated GEMM.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hc {

constexpr int kPBM = 128;   // tokens per tile (UMMA M, TMEM lanes)
constexpr int kPBN = 256;   // weight rows per tile (UMMA N, TMEM columns)
constexpr int kPBK = 64;    // K per pipeline stage (one 128-byte swizzle row of fp16)
constexpr int kPStages = 3;

// C[m][n] = Σ_k A[m][k]·B[n][k]  (+ Σ_j A2[m][j]·B2[n][j])   fp16 operands, fp32 accumulate in TMEM
struct PArgs {
  int M, N, K;          // tokens, output columns (weight rows), reduction length (K % 64 == 0)
  int K2;               // rank-slice reduction length (multiple of 16, <= 256), 0 = none
  int n_dim;            // UMMA N of this launch (multiple of 16, <= 256)
  int b_mode;           // 0: B = dequantised 4-bit weights (prefill codes); 1: B by TMA (fp16)
  const uint16_t* scales_t; // bf16 [K/128][N]  (b_mode 0; transposed so a stage reads 256 contiguous)
  const uint8_t* zeros_t;   // [K/128][N]
  int ksplit;               // split-K factor (>= 1); partial sums go to out + ks·M·ldo (fp32 only)
  void* out;
  int ldo;                  // row stride of out (elements)
  int out_type;             // 0 fp32, 1 bf16, 2 fp16
  int tiles_m, tiles_n;
  const float* rsig;        // optional [M] per-row factors 2^σ_m of the X prescale (launch_x_rows_f16), else NULL
};

// tmC: 2-D u32 tensor map over the nibble-paired codes [N][K/8] (box 8 words x 256 rows), b_mode 0.
cudaError_t launch_prefill(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA2,
                           const CUtensorMap& tmB2, const CUtensorMap& tmC, const PArgs& p, cudaStream_t st);
// Σ_ks partial[ks][m][0..n) -> fp16 out[m][0..ld) (deterministic split-K reduction)
cudaError_t launch_splitk_reduce_f16(const float* partial, int ksplit, int M, int ld, uint16_t* out, cudaStream_t st);
bool encode_tmap_codes(CUtensorMap* map, const void* base, uint64_t words_per_row, uint64_t rows);
// [rows][G] -> [G][rows] transposes of the per-group scales (bf16) and zeros (u8)
cudaError_t launch_transpose_groups(const uint16_t* s_in, const uint8_t* z_in, int rows, int G, uint16_t* s_out,
                                    uint8_t* z_out, cudaStream_t st);

// X bf16 [M][K] -> fp16 X' = X·2^-σ_m with a per-row power-of-two prescale; rsig[m] = 2^σ_m
cudaError_t launch_x_rows_f16(const uint16_t* in, int M, int K, uint16_t* out, float* rsig, cudaStream_t st);
// bf16 [n] -> fp16 [n]
cudaError_t launch_bf16_to_f16(const uint16_t* in, uint16_t* out, size_t n, cudaStream_t st);
// canonical 4-bit codes [rows][K/8] -> prefill nibble order (word w: nibbles k0,k2,k4,k6,k1,k3,k5,k7)
cudaError_t launch_prefill_codes(const uint32_t* canon, uint32_t* out, size_t n_words, cudaStream_t st);

// Encode a 2-D fp16 tensor map (row-major [outer][inner], row stride ld elements) with a
// 64 x box_rows box and 128-byte swizzle.  Returns false on failure.
bool encode_tmap_f16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                     uint32_t box_rows);

}  // namespace hc
