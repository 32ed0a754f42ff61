// Int8 tensor-core path of the decode kernel (2- and 4-bit codes, B <= 2; DESIGN.md §7.1 "I8").
//
// The fp16 path spends one lop3 + one hsub2 per two weights (plus shifts) turning codes into fp16
// A-fragments, which makes the decode loop ALU-bound well below HBM speed.  Here:
//  * A = the codes themselves as u8: with the 4-bit record layout of layout.h every byte of a code
//    word holds one code of row gid (low nibble) and one of row gid + 8 (high nibble), so
//    `w & 0x0F0F0F0F` is a row-gid u8 fragment and `w & 0xF0F0F0F0` a row-(gid + 8) fragment holding
//    16·q — one lop3 per four weights, no shift, no zero subtraction.  2-bit: the four 2-bit fields
//    of a byte are (row gid, row gid + 8) x (k block 8tig + 0..3, + 4..7) with weights 1, 4, 16, 64;
//    the x16 fields run as separate mma steps and join as acc1 + (acc2 >> 4) (exact);
//  * B = x in block fixed point: per (group, batch row) x_int = rint(x · 2^(29 − e)) with e the
//    exponent of the group's largest |x| (exact for every x within 2^22 of it), split into four
//    balanced base-256 digits (s8); mma column n = 4·b + d holds digit d of batch row b;
//  * mma.sync m16n8k32 u8·s8 accumulates Σ_k q·digit exactly in int32; the zero point is applied
//    exactly in integers (Σ (q − z)·digit = Σ q·digit − z·Σ digit, the digit sums precomputed);
//  * per record, each lane folds its two digit columns into one int (c_lo + 256·c_hi, |·| < 2^31),
//    converts once and accumulates s · 2^(16p + e − 29) · value in fp32 (one rounding per record,
//    like the fp16 path's per-group scale step);
//  * after the last record of an item the digit partials of a batch row are summed across the two
//    lanes holding them (fixed order: deterministic).
// x8 (shared memory, per group: x8_stride(B) = 544 B at B = 1, 1056 B at B = 2):
//   [n < 4B][tig 0..3][8 x u32]  B fragments: reg 2s + h = b_h of k32-step s, bytes = digit n&3 of
//                                 batch n>>2 at k = 32s + 8tig + 4h + {0, 2, 1, 3}
//   [tig < 2B] {int DD, float f} at 512·B: DD = D_(2p) + 256·D_(2p+1) (D_d = Σ_k digit_d of batch
//                                 b), f = 2^(16p + e_b − 29), for b = tig >> 1, p = tig & 1
// At B = 1 the lanes of batch-1 columns read whatever follows (their results are discarded); the
// region carries kX8Pad bytes of slack after the last group for them.
#pragma once
#include <stdint.h>

#include "decode_dev.cuh"

namespace hc {

__host__ __device__ __forceinline__ int x8_stride(int B) { return B == 1 ? 544 : 1056; }
constexpr int kX8Pad = 512;

__device__ __forceinline__ void imma16832(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ float pow2f(int e) { return __uint_as_float((uint32_t)(127 + e) << 23); }

// Stage x (bf16, global / L2) of groups [g0, g1) as x8 (a tile warp stages exactly the groups of its
// own item shares, warp_share, so it needs no barrier with the other warps).  Lane l holds
// k = 4l .. 4l + 3 of one (group, batch row).
__device__ __forceinline__ void x8_stage(const DArgs& a, uint8_t* x8, int g0, int g1, int lane) {
  const int tig = (lane >> 1) & 3, s = lane >> 3, h = lane & 1;
#ifndef HC_X8PRE
#define HC_X8PRE 4
#endif
  constexpr int kPre = HC_X8PRE;   // pieces whose loads are in flight together (round 2: 4 measured C2 r = 0 794 -> 817, C5 110.9 -> 112.6, C2 at allocated ranks ±0; round 1: 8 slower)
  for (int p0 = g0 * a.B; p0 < g1 * a.B; p0 += kPre) {
    // issue every load of the batch first: the staging is on the window's critical path and each load
    // is an L2 round trip (the x of this window was just written by its producer)
    uint2 rawv[kPre];
#pragma unroll
    for (int u = 0; u < kPre; ++u) {
      const int p = min(p0 + u, g1 * a.B - 1), g = a.B == 1 ? p : p >> 1, b = p - g * a.B;
      rawv[u] = __ldcg(reinterpret_cast<const uint2*>(a.x + (size_t)b * a.ldx + g * kGroup + 4 * lane));
    }
#pragma unroll
  for (int uu = 0; uu < kPre; ++uu) {
    const int p = p0 + uu;
    if (p >= g1 * a.B) break;
    const int g = a.B == 1 ? p : p >> 1, b = p - g * a.B;   // the int8 path runs B <= 2
    const uint2 raw = rawv[uu];
    const uint32_t hb[4] = {raw.x & 0xFFFFu, raw.x >> 16, raw.y & 0xFFFFu, raw.y >> 16};
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) m = max(m, hb[i] & 0x7FFFu);
    m = __reduce_max_sync(0xFFFFFFFFu, m);
#if HC_DEC_TRACE
    if (uu == 0 && p0 == g0 * a.B && lane == 0 && (threadIdx.x >> 5) == 0) {
      unsigned long long tt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
      if (g_dtrace) g_dtrace[((size_t)a.trace_slot * 512 + blockIdx.x) * 16 + 8] = tt;
    }
#endif
    // exponent of the group's largest |x|, clamped so that 2^(16p + e − 29) stays a normal float
    // (groups below 2^-97 keep 29 bits of fixed point relative to 2^-97).  A non-finite x (inf / NaN
    // bits, m >= 0x7F80) makes the group's scale NaN, so every output of the row is NaN (the float64
    // product with an inf or NaN operand and a zero weight is NaN too).
    const bool nonfinite = m >= 0x7F80u;
    const int e = (m == 0 || nonfinite) ? 0 : max(max((int)(m >> 7), 1) - 127, -97);
    const int sh = 29 - e, sh1 = sh >> 1;
    const float p1 = pow2f(sh1), p2 = pow2f(sh - sh1);     // 2^(29 − e) in two exact steps
    uint32_t u[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      u[i] = (uint32_t)__float2int_rn(__uint_as_float(hb[i] << 16) * p1 * p2) + 0x80808080u;   // balanced digits + 128
    uint8_t* blk = x8 + (size_t)g * x8_stride(a.B);
    int dsum[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const uint32_t sel = (uint32_t)d | ((uint32_t)(4 + d) << 4);
      const uint32_t t = prmt(u[0], u[1], sel), v = prmt(u[2], u[3], sel);
      const uint32_t reg = prmt(t, v, 0x5140u) ^ 0x80808080u;   // [u0.d, u2.d, u1.d, u3.d] − 128 each
      reinterpret_cast<uint32_t*>(blk)[((4 * b + d) * 4 + tig) * 8 + 2 * s + h] = reg;
      // Σ of this lane's four digits d: the s8 bytes of reg (one dp4a with ones instead of 4 extract-adds)
      dsum[d] = __reduce_add_sync(0xFFFFFFFFu, __dp4a((int)reg, 0x01010101, 0));
    }
    if (lane < 2) {
      const int pp = lane;
      int2 v;
      v.x = pp ? dsum[2] + 256 * dsum[3] : dsum[0] + 256 * dsum[1];
      v.y = nonfinite ? 0x7FC00000 : __float_as_int(pow2f(16 * pp + e - 29));
      reinterpret_cast<int2*>(blk + 512 * a.B)[2 * b + pp] = v;
    }
  }
  }
}

// One (row-block, group) record on the int8 path: tot[0] += row gid, tot[2] += row gid + 8 partial
// of this lane's two digit columns (tot[1], tot[3] unused until i8_finish).  dd_off = 512·B.
template <int BITS>
__device__ __forceinline__ void i8_tile(const uint8_t* rec, int lane, const uint8_t* x8g, int dd_off,
                                        float (&tot)[1][4]) {
  static_assert(BITS == 2 || BITS == 4, "int8 path: 2- or 4-bit codes");
  const int gid = lane >> 2, tig = lane & 3;
  const uint32_t sw = *reinterpret_cast<const uint32_t*>(rec + scales_off(BITS) + 4 * gid);
  const uint2 zz = *reinterpret_cast<const uint2*>(rec + zeros_off(BITS));
  // digit rows 4b + d exist for b < B only (dd_off = 512·B): the columns of lanes beyond them are discarded,
  // so those lanes read row 0 of the same group instead of the next group's bytes (no cross-warp read)
  const int gid_r = min(gid, (dd_off >> 7) - 1);
  const uint4* xb = reinterpret_cast<const uint4*>(x8g) + (gid_r * 4 + tig) * 2;
  const uint4 bv0 = xb[0], bv1 = xb[1];
  const uint32_t bb[8] = {bv0.x, bv0.y, bv0.z, bv0.w, bv1.x, bv1.y, bv1.z, bv1.w};
  const int2 ddf = reinterpret_cast<const int2*>(x8g + dd_off)[tig];
  int c[4] = {0, 0, 0, 0};
  if constexpr (BITS == 4) {
    const uint4 w0 = *reinterpret_cast<const uint4*>(rec + lane * 16);
    const uint4 w1 = *reinterpret_cast<const uint4*>(rec + 512 + lane * 16);
    const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
    for (int s = 0; s < 4; ++s)
      imma16832(c, w[2 * s] & 0x0F0F0F0Fu, w[2 * s] & 0xF0F0F0F0u, w[2 * s + 1] & 0x0F0F0F0Fu,
                w[2 * s + 1] & 0xF0F0F0F0u, bb[2 * s], bb[2 * s + 1]);
  } else {
    const uint4 wv = *reinterpret_cast<const uint4*>(rec + lane * 16);
    const uint32_t w[4] = {wv.x, wv.y, wv.z, wv.w};
    int c2[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; q += 2) {
      imma16832(c, w[q] & 0x03030303u, w[q] & 0x0C0C0C0Cu, w[q + 1] & 0x03030303u, w[q + 1] & 0x0C0C0C0Cu,
                bb[2 * q], bb[2 * q + 2]);
      imma16832(c2, w[q] & 0x30303030u, w[q] & 0xC0C0C0C0u, w[q + 1] & 0x30303030u, w[q + 1] & 0xC0C0C0C0u,
                bb[2 * q + 1], bb[2 * q + 3]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) c[e] += c2[e] >> 4;    // the x16 fields: exact multiples of 16
  }
  constexpr int kHi = 1 << row_hi_shift(BITS);        // row gid + 8 weight: 16 (4-bit), 4 (2-bit)
  const int z0 = (int)((zz.x >> (4 * gid)) & 15u), z8 = (int)((zz.y >> (4 * gid)) & 15u);
  // modular int32 arithmetic: the results fit (|·| < 2^31), intermediates may wrap harmlessly
  const int v0 = (int)((uint32_t)c[0] + 256u * (uint32_t)c[1] - (uint32_t)(z0 * ddf.x));
  const int v8 = (int)((uint32_t)c[2] + 256u * (uint32_t)c[3] - (uint32_t)(kHi * z8 * ddf.x));
  const float f = __int_as_float(ddf.y);
  const float s0 = bf16_bits_to_f32(sw & 0xFFFFu) * f, s1 = bf16_bits_to_f32(sw >> 16) * (f * (1.f / kHi));
  tot[0][0] = fmaf(s0, (float)v0, tot[0][0]);
  tot[0][2] = fmaf(s1, (float)v8, tot[0][2]);
}

// End of an item: sum the digit-pair partials of each batch row (lanes tig 0+1: batch 0, 2+3:
// batch 1) and lay the result out like the fp16 path's fragments (lane tig 0: cols 0, 1).
__device__ __forceinline__ void i8_finish(float (&tot)[1][4], int lane, int B) {
  const int tig = lane & 3;
  float t0 = tot[0][0], t8 = tot[0][2];
  t0 += __shfl_xor_sync(0xFFFFFFFFu, t0, 1);
  t8 += __shfl_xor_sync(0xFFFFFFFFu, t8, 1);
  const float u0 = __shfl_down_sync(0xFFFFFFFFu, t0, 2), u8 = __shfl_down_sync(0xFFFFFFFFu, t8, 2);
  if (tig == 0) {
    tot[0][0] = t0; tot[0][1] = B > 1 ? u0 : 0.f; tot[0][2] = t8; tot[0][3] = B > 1 ? u8 : 0.f;
  } else {
    tot[0][0] = 0.f; tot[0][1] = 0.f; tot[0][2] = 0.f; tot[0][3] = 0.f;
  }
}

}  // namespace hc
