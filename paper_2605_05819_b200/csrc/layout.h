// Kernel-side HBM layout of one compensated linear (product code; NOT shared with oracle/).
//
// The C-ABI takes canonical formats (include/hcinfer.h); hc_load_layer repacks them
// once into the layout below, chosen so that the decode kernel
//   * streams every weight byte exactly once with 16-byte-aligned bulk (TMA) copies,
//   * turns each 32-bit code word into mma.sync A-fragment registers with at most one
//     shift per word plus one lop3 per register (the fp16 "magic number" trick:
//     0x6400 | field = 1024 + field, exact: fp16 has 10 mantissa bits),
//   * never materialises W.
//
// Row block (rb) = 16 output rows (the mma M dimension).  Group = 128 input
// elements (the quantisation group).  A lane of a warp owns,
// per (rb, group), the A-fragments of all eight k16 steps of the group:
//     lane = 4*gid + tig;  register (j, i), step j in 0..7, reg i in 0..3 holds
//     row  = gid + 8*(i&1)
//     k_lo = 32*(j>>1) + 8*tig + 4*(j&1) + 2*(i>>1),  k_hi = k_lo + 1   (k within the group)
// The k permutation is legal because the per-group partial sum is order-free; it makes
// lane tig's x values for steps (2q, 2q+1) one 16-byte run x[32q + 8tig .. +7].
//
// Record for (rb, group) = [codes: 32 lanes x 2*bits words][scales 8 x u32][zeros u64][pad 8]
//   codes word w of lane l at byte  (w/4)*512 + l*16 + (w%4)*4   for w < 4*(2b/4)
//                                   512*(2b/4) + l*8 + (w%4)*4    for the 2-word tail (b = 3)
//   scales word gid = bf16 s[row gid] | bf16 s[row gid+8] << 16
//   zeros  u64: row r's zero in bits [4r, 4r+4)
//
// Register extraction ("slots"): register (j, i) = 0x64006400 | field bits, where a
// field is up to 3 "parts" (word, shift, pos, nbits) taken from the lo 16-bit half
// (and the same bits +16 from the hi half).  The register then holds
// 1024 + q*2^fp in both halves (exact in fp16), fp = the field's bit position.  The B operand
// (x) of k pair p is pre-scaled by 2^-fp of the row-gid register (i = 2p): x' = x·2^-fp, exact in
// fp16 for normal-range x (R20).  The row gid + 8 register of the pair may sit
// row_hi_shift(bits) bits higher; its products are then 2^row_hi_shift too large and that row's
// group scale is divided by the same power of two (exact).
//   4-bit: word j, fields at bits [0,4) (fp 0, row gid) and [4,8) (fp 4, row gid + 8) of w and
//          of w >> 8 (k pairs 0 and 1); x' = x;
//   2-bit: word j/2, fields at bits 4(j&1) (fp 4(j&1), row gid) and 4(j&1) + 2 (row gid + 8) of w
//          and of w >> 8 (k pairs 0 and 1);
//   3-bit: fields at bits 0-2 and 3-5 (fp 3) of w >> {0, 6, 12}, plus two registers gathered
//          from bit 15 of the six words.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define HC_HD __host__ __device__ __forceinline__
#else
#define HC_HD inline
#endif

namespace hc {

constexpr int kRows = 16;
constexpr int kGroup = 128;
constexpr uint32_t kMagic = 0x64006400u;   // fp16x2(1024, 1024)
constexpr float kMagicF = 1024.f;

HC_HD constexpr int code_words(int bits) { return 2 * bits; }            // per lane per group
HC_HD constexpr int code_bytes(int bits) { return 256 * bits; }          // per (rb, group)
HC_HD constexpr int rec_bytes(int bits) { return 256 * bits + 48; }      // + scales/zeros/pad
HC_HD constexpr int scales_off(int bits) { return 256 * bits; }
HC_HD constexpr int zeros_off(int bits) { return 256 * bits + 32; }

HC_HD constexpr int word_offset(int bits, int w, int lane) {
  return (w < 4 * ((2 * bits) / 4))
             ? (w / 4) * 512 + lane * 16 + (w % 4) * 4
             : 512 * ((2 * bits) / 4) + lane * 8 + (w % 4) * 4;
}

struct Part { int word, shift, pos, nbits; };
struct Slot { int nparts; int fp; Part p[3]; };

// Slot table for register (j, i) at a given bit width.  See the header comment.
HC_HD constexpr Slot slot(int bits, int j, int i) {
  if (bits == 4) {
    // row gid (i even) <- the low nibbles of word j's bytes, row gid + 8 (i odd) <- the high
    // nibbles; k pair i>>1 <- bytes {0, 2} (shift 0) or {1, 3} (shift 8).  Each byte-wise half of
    // a word is one row's 4 codes, so `w & 0x0F0F0F0F` / `w & 0xF0F0F0F0` are u8 A-fragments of
    // the int8 mma path (decode_i8.cuh) and the fp16 path extracts with one lop3 per register.
    const int fp = 4 * (i & 1);
    return Slot{1, fp, {Part{j, 8 * (i >> 1), fp, 4}, Part{0, 0, 0, 0}, Part{0, 0, 0, 0}}};
  }
  if (bits == 2) {
    // word j/2; k pair i>>1 <- bytes {0, 2} (shift 0) or {1, 3} (shift 8); field 2·(j&1) + (i&1) of
    // each byte: row gid in fields 0 / 2, row gid + 8 in fields 1 / 3 (4x higher), so each field
    // mask (0x03030303 << 2f) of a word is a u8 A-fragment of the int8 path (decode_i8.cuh)
    const int fp = 4 * (j & 1) + 2 * (i & 1);
    return Slot{1, fp, {Part{j / 2, 8 * (i >> 1), fp, 2}, Part{0, 0, 0, 0}, Part{0, 0, 0, 0}}};
  }
  // bits == 3: 20 weight-1 slots (18 plain + 2 gathered from bit 15 of each word),
  // 12 weight-8 slots; steps 0..5 pair (w1, w8), steps 6..7 pair (w1, w1).
  const int pair = i >> 1, mem = i & 1;
  int w1 = -1, w8 = -1;
  if (j < 6) { if (pair == 0) w1 = 2 * j + mem; else w8 = 2 * j + mem; }
  else       { w1 = 12 + 4 * (j - 6) + 2 * pair + mem; }
  if (w8 >= 0) {
    return Slot{1, 3, {Part{w8 / 2, 6 * (w8 % 2), 3, 3}, Part{0, 0, 0, 0}, Part{0, 0, 0, 0}}};
  }
  if (w1 < 18) {
    return Slot{1, 0, {Part{w1 / 3, 6 * (w1 % 3), 0, 3}, Part{0, 0, 0, 0}, Part{0, 0, 0, 0}}};
  }
  const int base = (w1 == 18) ? 0 : 3;   // gather bit 15 of words base..base+2
  return Slot{3, 0, {Part{base, 15, 0, 1}, Part{base + 1, 14, 1, 1}, Part{base + 2, 13, 2, 1}}};
}

// Extra exponent of the row gid + 8 registers over the row gid registers of the same k pair.
HC_HD constexpr int row_hi_shift(int bits) { return bits == 4 ? 4 : (bits == 2 ? 2 : 0); }

// x pre-scale exponent for the B register of step j: pair 0 (b0, cols 2tig..) or pair 1 (b1).
HC_HD constexpr int step_fp(int bits, int j, int pair) { return slot(bits, j, 2 * pair).fp; }

// Fragment element -> (row within rb, k within group)
HC_HD constexpr int frag_row(int lane, int i) { return (lane >> 2) + 8 * (i & 1); }
// k within the group: 32*(j>>1) + 8*tig + 4*(j&1) + 2*(i>>1) + hi.  For a fixed pair of steps
// (2q, 2q+1) the four tig lanes of a row read one contiguous 64 B run of x (16 B each), so
// 128-bit x loads are conflict-free in shared memory and fully coalesced in global memory.
HC_HD constexpr int frag_k(int lane, int j, int i, int hi) {
  return 32 * (j >> 1) + 8 * (lane & 3) + 4 * (j & 1) + 2 * (i >> 1) + hi;
}

// Compensation factor tiles (bf16, no quantisation):
//  U: [rb][chunk c = rank/16][lane][uint4]; reg i of lane: row gid + 8(i&1), ranks 16c + 2tig + 8(i>>1) + {0,1}
//  V: [chunk c][group g][step j][lane][uint4]; reg i: rank 16c + gid + 8(i&1), k = frag_k(lane, j, i, {0,1})
HC_HD constexpr int u_rank(int lane, int i, int hi) { return 2 * (lane & 3) + 8 * (i >> 1) + hi; }

}  // namespace hc
