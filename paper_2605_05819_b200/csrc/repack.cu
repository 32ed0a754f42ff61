// Load-time repack (hc_load_layer) and its host test exports.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "hcinfer.h"
#include "repack.cuh"
#include "repack_kernels.h"
#include "status.h"

namespace hc {

// one thread per (rb, g, lane)
__global__ void repack_codes_kernel(RepackSrc src, int n_rb, int K, int bits, uint8_t* __restrict__ out) {
  const int G = K / kGroup;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)n_rb * G * 32;
  if (tid >= total) return;
  const int lane = (int)(tid & 31);
  const long long rg = tid >> 5;
  const int g = (int)(rg % G), rb = (int)(rg / G);
  const int wpr = K * bits / 32;
  uint32_t words[8];
  pack_lane_words(src.codes[0], src.codes[1], src.rstride, wpr, rb, g, lane, bits, words);
  uint8_t* rec = out + (size_t)rg * rec_bytes(bits);
  for (int w = 0; w < 2 * bits; ++w) *reinterpret_cast<uint32_t*>(rec + word_offset(bits, w, lane)) = words[w];
  if (lane < 8) {
    const uint16_t s0 = row_ptr(src.scales[0], src.scales[1], src.rstride, (size_t)G, rb, lane)[g];
    const uint16_t s1 = row_ptr(src.scales[0], src.scales[1], src.rstride, (size_t)G, rb, lane + 8)[g];
    *reinterpret_cast<uint32_t*>(rec + scales_off(bits) + 4 * lane) = (uint32_t)s0 | ((uint32_t)s1 << 16);
  }
  if (lane == 8) {
    uint64_t zw = 0;
    for (int r = 0; r < kRows; ++r)
      zw |= (uint64_t)(row_ptr(src.zeros[0], src.zeros[1], src.rstride, (size_t)G, rb, r)[g] & 0xF) << (4 * r);
    *reinterpret_cast<uint64_t*>(rec + zeros_off(bits)) = zw;
    *reinterpret_cast<uint64_t*>(rec + zeros_off(bits) + 8) = 0ull;
  }
}

// U: [rb][c][lane][4 regs]; one thread per (rb, c, lane)
__global__ void repack_u_kernel(RepackSrc src, int n_rb, int r_stored, uint32_t* __restrict__ out) {
  const int nc = r_stored / 16;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)n_rb * nc * 32) return;
  const int lane = (int)(tid & 31);
  const int c = (int)((tid >> 5) % nc), rb = (int)((tid >> 5) / nc);
  for (int i = 0; i < 4; ++i) {
    const uint16_t* row = row_ptr(src.U[0], src.U[1], src.rstride, (size_t)r_stored, rb, frag_row(lane, i));
    const uint32_t lo = row[16 * c + u_rank(lane, i, 0)];
    const uint32_t hi = row[16 * c + u_rank(lane, i, 1)];
    out[tid * 4 + i] = lo | (hi << 16);
  }
}

// V: [c][g][j][lane][4 regs]; one thread per (c, g, j, lane)
__global__ void repack_v_kernel(const uint16_t* __restrict__ V, int K, int r_stored, uint32_t* __restrict__ out) {
  const int G = K / kGroup, nc = r_stored / 16;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)nc * G * 8 * 32) return;
  const int lane = (int)(tid & 31);
  const int j = (int)((tid >> 5) & 7);
  const long long cg = tid >> 8;
  const int g = (int)(cg % G), c = (int)(cg / G);
  for (int i = 0; i < 4; ++i) {
    const size_t rank = (size_t)(16 * c + frag_row(lane, i));
    const uint32_t lo = V[rank * K + g * kGroup + frag_k(lane, j, i, 0)];
    const uint32_t hi = V[rank * K + g * kGroup + frag_k(lane, j, i, 1)];
    out[tid * 4 + i] = lo | (hi << 16);
  }
}

// Vn: [kb][c][lane][4 regs]; reg i of lane: rank 16c + gid + 8(i&1), k = 16kb + 2tig + 8(i>>1) + {0,1}
// (k-block major: the chunks of one 16-k block are contiguous, one bulk copy per member)
__global__ void repack_vn_kernel(const uint16_t* __restrict__ V, int K, int r_stored, uint32_t* __restrict__ out) {
  const int KB = K / 16, nc = r_stored / 16;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)nc * KB * 32) return;
  const int lane = (int)(tid & 31);
  const long long ck = tid >> 5;
  const int c = (int)(ck % nc), kb = (int)(ck / nc);
  for (int i = 0; i < 4; ++i) {
    const size_t rank = (size_t)(16 * c + (lane >> 2) + 8 * (i & 1));
    const int k = 16 * kb + 2 * (lane & 3) + 8 * (i >> 1);
    out[tid * 4 + i] = (uint32_t)V[rank * K + k] | ((uint32_t)V[rank * K + k + 1] << 16);
  }
}

cudaError_t launch_repack_vn(const uint16_t* V, int K, int r_stored, uint32_t* out, cudaStream_t st) {
  if (r_stored <= 0) return cudaSuccess;
  const long long n = (long long)(r_stored / 16) * (K / 16) * 32;
  repack_vn_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(V, K, r_stored, out);
  return cudaGetLastError();
}

cudaError_t launch_repack_records(const RepackSrc& src, int K, int bits, int r_stored, int n_rb, uint8_t* rec_out,
                                  uint32_t* u_out, cudaStream_t st) {
  const int G = K / kGroup;
  long long n = (long long)n_rb * G * 32;
  repack_codes_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, n_rb, K, bits, rec_out);
  if (r_stored > 0) {
    n = (long long)n_rb * (r_stored / 16) * 32;
    repack_u_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(src, n_rb, r_stored, u_out);
  }
  return cudaGetLastError();
}

// ---- fp8 (e4m3) compensation factors: the same fragment orders, one byte per value.
// NaN encodings (|b| = 0x7F) raise *nan_flag.
// U8: [rb][c][lane][8 bytes], byte 2i + h = U[row frag_row(lane, i)][16c + u_rank(lane, i, h)]
__global__ void repack_u8_kernel(const uint8_t* __restrict__ U0, const uint8_t* __restrict__ U1, int rstride, int n_rb,
                                 int r_stored, uint8_t* __restrict__ out, unsigned* nan_flag) {
  const int nc = r_stored / 16;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)n_rb * nc * 32) return;
  const int lane = (int)(tid & 31);
  const int c = (int)((tid >> 5) % nc), rb = (int)((tid >> 5) / nc);
  unsigned bad = 0;
  for (int i = 0; i < 4; ++i) {
    const uint8_t* row = row_ptr(U0, U1, rstride, (size_t)r_stored, rb, frag_row(lane, i));
    for (int h = 0; h < 2; ++h) {
      const uint8_t b = row[16 * c + u_rank(lane, i, h)];
      bad |= (b & 0x7Fu) == 0x7Fu;
      out[tid * 8 + 2 * i + h] = b;
    }
  }
  if (bad) atomicOr(nan_flag, 1u);
}
// V8 pieces: [c][g][j][lane][8 bytes] (j = step), byte 2i + h = V[rank 16c + frag_row(lane, i)][g·128 + frag_k(lane, j, i, h)];
// one 1 KB piece = steps 4p .. 4p + 3 of a (chunk, group) = 16 ranks x 64 k
__global__ void repack_v8_kernel(const uint8_t* __restrict__ V, int K, int r_stored, uint8_t* __restrict__ out,
                                 unsigned* nan_flag) {
  const int G = K / kGroup, nc = r_stored / 16;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)nc * G * 8 * 32) return;
  const int lane = (int)(tid & 31);
  const int j = (int)((tid >> 5) & 7);
  const long long cg = tid >> 8;
  const int g = (int)(cg % G), c = (int)(cg / G);
  unsigned bad = 0;
  for (int i = 0; i < 4; ++i) {
    const size_t rank = (size_t)(16 * c + frag_row(lane, i));
    for (int h = 0; h < 2; ++h) {
      const uint8_t b = V[rank * K + g * kGroup + frag_k(lane, j, i, h)];
      bad |= (b & 0x7Fu) == 0x7Fu;
      out[tid * 8 + 2 * i + h] = b;
    }
  }
  if (bad) atomicOr(nan_flag, 1u);
}

// e4m3 -> float: the byte's magnitude bits placed as a bf16 (exponent field e, mantissa m << 4) is the value
// times 2^-120 for normals and subnormals alike; x 2^120 is exact.
__device__ __forceinline__ float e4m3_to_f32(uint8_t b) {
  const uint32_t bits = ((uint32_t)(b & 0x7Fu) << 20) | ((uint32_t)(b & 0x80u) << 24);
  return __uint_as_float(bits) * 0x1p120f;
}

// Prefill copies of fp8 factors: out[i] = fp16(e4m3(in[i]) · scale[rank of i]); rank = i / per_rank (V rows) or
// i % r_stored (U rows).
__global__ void fp8_to_f16_kernel(const uint8_t* __restrict__ in, const float* __restrict__ scale, size_t n, int r_stored,
                                  int rank_major, int K, uint16_t* __restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int rank = rank_major ? (int)(i / (size_t)K) : (int)(i % (size_t)r_stored);
  out[i] = __half_as_ushort(__float2half_rn(e4m3_to_f32(in[i]) * scale[rank]));
}

cudaError_t launch_repack_fp8(const uint8_t* U0, const uint8_t* U1, int rstride, int n_rb, const uint8_t* V, int K,
                              int r_stored, uint8_t* u_out, uint8_t* v_out, unsigned* nan_flag, cudaStream_t st) {
  if (r_stored <= 0) return cudaSuccess;
  if (u_out && n_rb > 0) {
    const long long nu = (long long)n_rb * (r_stored / 16) * 32;
    repack_u8_kernel<<<(unsigned)((nu + 255) / 256), 256, 0, st>>>(U0, U1, rstride, n_rb, r_stored, u_out, nan_flag);
  }
  if (v_out) {
    const long long nv = (long long)(r_stored / 16) * (K / kGroup) * 8 * 32;
    repack_v8_kernel<<<(unsigned)((nv + 255) / 256), 256, 0, st>>>(V, K, r_stored, v_out, nan_flag);
  }
  return cudaGetLastError();
}

cudaError_t launch_fp8_to_f16(const uint8_t* in, const float* scale, size_t n, int r_stored, bool rank_major, int K,
                              uint16_t* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  fp8_to_f16_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, scale, n, r_stored, rank_major ? 1 : 0, K, out);
  return cudaGetLastError();
}

// ---- inverse repack on the device (lazy prefill copies, built on the first B > 16 call from the decode
// records and factor fragments instead of being kept from load time)
// records [n_rb][G][rec] -> q bytes [rows][K], scales bf16 [rows][G], zeros [rows][G]; one thread per (rb, g, lane)
__global__ void unrepack_records_kernel(const uint8_t* __restrict__ rec, int n_rb, int K, int bits, uint8_t* __restrict__ q,
                                        uint16_t* __restrict__ scales, uint8_t* __restrict__ zeros) {
  const int G = K / kGroup;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)n_rb * G * 32) return;
  const int lane = (int)(tid & 31);
  const long long rg = tid >> 5;
  const int g = (int)(rg % G), rb = (int)(rg / G);
  const uint8_t* r = rec + (size_t)rg * rec_bytes(bits);
  uint32_t words[8];
  for (int w = 0; w < 2 * bits; ++w) words[w] = *reinterpret_cast<const uint32_t*>(r + word_offset(bits, w, lane));
  unpack_lane_words(words, lane, bits, g, rb, q, K);
  if (lane < 8) {
    const uint32_t sw = *reinterpret_cast<const uint32_t*>(r + scales_off(bits) + 4 * lane);
    scales[((size_t)rb * kRows + lane) * G + g] = (uint16_t)(sw & 0xFFFFu);
    scales[((size_t)rb * kRows + lane + 8) * G + g] = (uint16_t)(sw >> 16);
  }
  if (lane == 8) {
    const uint64_t zw = *reinterpret_cast<const uint64_t*>(r + zeros_off(bits));
    for (int rr = 0; rr < kRows; ++rr) zeros[((size_t)rb * kRows + rr) * G + g] = (uint8_t)((zw >> (4 * rr)) & 0xF);
  }
}
// q bytes [n][K] -> canonical 4-bit code words [n][K/8] (element k at bits 4k)
__global__ void pack4_kernel(const uint8_t* __restrict__ q, size_t n_words, uint32_t* __restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_words) return;
  const uint2 v = *reinterpret_cast<const uint2*>(q + 8 * i);
  uint32_t w = 0;
  for (int j = 0; j < 4; ++j) w |= ((v.x >> (8 * j)) & 0xFu) << (4 * j);
  for (int j = 0; j < 4; ++j) w |= ((v.y >> (8 * j)) & 0xFu) << (16 + 4 * j);
  out[i] = w;
}
__device__ __forceinline__ float frag_val(const uint8_t* base, size_t reg, int h, const float* scale, int rank) {
  if (scale) {                                           // fp8: e4m3 byte 2i + h, times the rank's scale
    const uint8_t b = base[reg * 2 + h];
    return e4m3_to_f32(b) * scale[rank];
  }
  const uint32_t v = reinterpret_cast<const uint32_t*>(base)[reg];
  return __uint_as_float((h ? (v >> 16) : (v & 0xFFFFu)) << 16);
}
// U fragments [rb][c][lane][4 regs] -> fp16 U [rows][r_stored]; fp8: the e4m3 bytes x u_scale
__global__ void unrepack_u_f16_kernel(const uint8_t* __restrict__ U, int n_rb, int r_stored, const float* __restrict__ us,
                                      uint16_t* __restrict__ out) {
  const int nc = r_stored / 16;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)n_rb * nc * 32) return;
  const int lane = (int)(tid & 31);
  const int c = (int)((tid >> 5) % nc), rb = (int)((tid >> 5) / nc);
  for (int i = 0; i < 4; ++i)
    for (int h = 0; h < 2; ++h) {
      const int row = rb * kRows + frag_row(lane, i), rank = 16 * c + u_rank(lane, i, h);
      out[(size_t)row * r_stored + rank] = __half_as_ushort(__float2half_rn(frag_val(U, (size_t)tid * 4 + i, h, us, rank)));
    }
}
// V fragments [c][g][j][lane][4 regs] -> fp16 V [r_stored][K]; fp8: x v_scale
__global__ void unrepack_v_f16_kernel(const uint8_t* __restrict__ V, int K, int r_stored, const float* __restrict__ vs,
                                      uint16_t* __restrict__ out) {
  const int G = K / kGroup, nc = r_stored / 16;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid >= (long long)nc * G * 8 * 32) return;
  const int lane = (int)(tid & 31);
  const int j = (int)((tid >> 5) & 7);
  const long long cg = tid >> 8;
  const int g = (int)(cg % G), c = (int)(cg / G);
  for (int i = 0; i < 4; ++i)
    for (int h = 0; h < 2; ++h) {
      const int rank = 16 * c + frag_row(lane, i);
      const int k = g * kGroup + frag_k(lane, j, i, h);
      out[(size_t)rank * K + k] = __half_as_ushort(__float2half_rn(frag_val(V, (size_t)tid * 4 + i, h, vs, rank)));
    }
}

cudaError_t launch_unrepack_prefill(const uint8_t* rec, int n_rb, int K, int bits, uint8_t* q_tmp, uint32_t* codes_out,
                                    uint16_t* scales_out, uint8_t* zeros_out, const uint8_t* Ufrag, const uint8_t* Vfrag,
                                    int r_stored, const float* us, const float* vs, uint16_t* U16, uint16_t* V16,
                                    cudaStream_t st) {
  const long long n = (long long)n_rb * (K / kGroup) * 32;
  unrepack_records_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rec, n_rb, K, bits, q_tmp, scales_out, zeros_out);
  const size_t nw = (size_t)n_rb * kRows * K / 8;
  pack4_kernel<<<(unsigned)((nw + 255) / 256), 256, 0, st>>>(q_tmp, nw, codes_out);
  if (r_stored > 0) {
    const long long nu = (long long)n_rb * (r_stored / 16) * 32;
    unrepack_u_f16_kernel<<<(unsigned)((nu + 255) / 256), 256, 0, st>>>(Ufrag, n_rb, r_stored, us, U16);
    const long long nv = (long long)(r_stored / 16) * (K / kGroup) * 8 * 32;
    unrepack_v_f16_kernel<<<(unsigned)((nv + 255) / 256), 256, 0, st>>>(Vfrag, K, r_stored, vs, V16);
  }
  return cudaGetLastError();
}

cudaError_t launch_repack_v(const uint16_t* V, int K, int r_stored, uint32_t* v_out, cudaStream_t st) {
  if (r_stored <= 0) return cudaSuccess;
  const long long n = (long long)(r_stored / 16) * (K / kGroup) * 8 * 32;
  repack_v_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(V, K, r_stored, v_out);
  return cudaGetLastError();
}

}  // namespace hc

// ------------------------------------------------------------------ host test exports
extern "C" size_t hc_repacked_bytes(int32_t N, int32_t K, int32_t bits) {
  if (N <= 0 || K <= 0 || N % hc::kRows || K % hc::kGroup) return 0;
  return (size_t)(N / hc::kRows) * (K / hc::kGroup) * hc::rec_bytes(bits);
}

static bool bits_ok(int b) { return b == 2 || b == 3 || b == 4; }

extern "C" hc_status hc_repack_host(const uint32_t* codes, const uint16_t* scales, const uint8_t* zeros,
                                    int32_t N, int32_t K, int32_t bits, uint8_t* out) {
  using namespace hc;
  if (!codes || !scales || !zeros || !out) return fail(HC_ERR_CONFIG, "hc_repack_host: null pointer");
  if (!bits_ok(bits) || N <= 0 || N % kRows || K <= 0 || K % kGroup)
    return fail(HC_ERR_CONFIG, "hc_repack_host: bad shape N=%d K=%d bits=%d", N, K, bits);
  const int G = K / kGroup, wpr = K * bits / 32;
  for (int rb = 0; rb < N / kRows; ++rb)
    for (int g = 0; g < G; ++g) {
      uint8_t* rec = out + ((size_t)rb * G + g) * rec_bytes(bits);
      std::memset(rec, 0, rec_bytes(bits));
      for (int lane = 0; lane < 32; ++lane) {
        uint32_t words[8];
        pack_lane_words(codes, codes + (size_t)8 * wpr, kRows, wpr, rb, g, lane, bits, words);
        for (int w = 0; w < 2 * bits; ++w) std::memcpy(rec + word_offset(bits, w, lane), &words[w], 4);
      }
      for (int gid = 0; gid < 8; ++gid) {
        const size_t r0 = (size_t)rb * kRows + gid;
        const uint32_t sw = (uint32_t)scales[r0 * G + g] | ((uint32_t)scales[(r0 + 8) * G + g] << 16);
        std::memcpy(rec + scales_off(bits) + 4 * gid, &sw, 4);
      }
      uint64_t zw = 0;
      for (int r = 0; r < kRows; ++r) zw |= (uint64_t)(zeros[((size_t)rb * kRows + r) * G + g] & 0xF) << (4 * r);
      std::memcpy(rec + zeros_off(bits), &zw, 8);
    }
  return HC_OK;
}

extern "C" hc_status hc_unpack_repacked_host(const uint8_t* packed, int32_t N, int32_t K, int32_t bits,
                                             uint8_t* q_out, uint16_t* scales_out, uint8_t* zeros_out) {
  using namespace hc;
  if (!packed || !q_out) return fail(HC_ERR_CONFIG, "hc_unpack_repacked_host: null pointer");
  if (!bits_ok(bits) || N <= 0 || N % kRows || K <= 0 || K % kGroup)
    return fail(HC_ERR_CONFIG, "hc_unpack_repacked_host: bad shape");
  const int G = K / kGroup;
  for (int rb = 0; rb < N / kRows; ++rb)
    for (int g = 0; g < G; ++g) {
      const uint8_t* rec = packed + ((size_t)rb * G + g) * rec_bytes(bits);
      for (int lane = 0; lane < 32; ++lane) {
        uint32_t words[8];
        for (int w = 0; w < 2 * bits; ++w) std::memcpy(&words[w], rec + word_offset(bits, w, lane), 4);
        unpack_lane_words(words, lane, bits, g, rb, q_out, K);
      }
      if (scales_out)
        for (int gid = 0; gid < 8; ++gid) {
          uint32_t sw;
          std::memcpy(&sw, rec + scales_off(bits) + 4 * gid, 4);
          scales_out[((size_t)rb * kRows + gid) * G + g] = (uint16_t)(sw & 0xFFFF);
          scales_out[((size_t)rb * kRows + gid + 8) * G + g] = (uint16_t)(sw >> 16);
        }
      if (zeros_out) {
        uint64_t zw;
        std::memcpy(&zw, rec + zeros_off(bits), 8);
        for (int r = 0; r < kRows; ++r) zeros_out[((size_t)rb * kRows + r) * G + g] = (uint8_t)((zw >> (4 * r)) & 0xF);
      }
    }
  return HC_OK;
}
