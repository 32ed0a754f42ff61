// Canonical C-ABI formats -> kernel records (layout.h).  __host__ __device__ so the same
// mapping runs in the load-time repack kernel and in the host test exports.
#pragma once
#include <stdint.h>

#include "layout.h"

namespace hc {

// unsigned code q[n][k] from the canonical little-endian bitstream of row n
HC_HD uint32_t canon_code(const uint32_t* row, int k, int bits) {
  const int p = bits * k, w = p >> 5, off = p & 31;
  uint32_t v = row[w] >> off;
  if (off + bits > 32) v |= row[w + 1] << (32 - off);
  return v & ((1u << bits) - 1u);
}

// Row r (0..15) of row block rb comes from `lo` (r < 8) or `hi` (r >= 8), source row
// rb*rstride + (r & 7).  Plain matrices: lo = rows, hi = rows + 8 rows, rstride = 16.
// Fused SiLU(gate)·up windows: lo = up, hi = gate, rstride = 8 (row blocks interleave 8 + 8 rows).
template <typename T>
HC_HD const T* row_ptr(const T* lo, const T* hi, int rstride, size_t row_elems, int rb, int r) {
  return (r < 8 ? lo : hi) + ((size_t)rb * rstride + (r & 7)) * row_elems;
}

// The 2*bits code words of lane `lane` for record (rb, g).
// codes: canonical [N][K*bits/32] (row stride `wpr` words).
HC_HD void pack_lane_words(const uint32_t* lo, const uint32_t* hi, int rstride, int wpr, int rb, int g, int lane,
                           int bits, uint32_t* out /* [2*bits] */) {
  for (int w = 0; w < 2 * bits; ++w) out[w] = 0u;
  for (int j = 0; j < 8; ++j) {
    for (int i = 0; i < 4; ++i) {
      const Slot s = slot(bits, j, i);
      const uint32_t* r = row_ptr(lo, hi, rstride, (size_t)wpr, rb, frag_row(lane, i));
      for (int h = 0; h < 2; ++h) {
        const int k = g * kGroup + frag_k(lane, j, i, h);
        const uint32_t val = canon_code(r, k, bits) << s.fp;   // field value in the 16-bit half
        for (int p = 0; p < s.nparts; ++p) {
          const Part& pt = s.p[p];
          const uint32_t bitsv = (val >> pt.pos) & ((1u << pt.nbits) - 1u);
          out[pt.word] |= bitsv << (pt.shift + pt.pos + 16 * h);
        }
      }
    }
  }
}

// Inverse: decode lane words back to q for the 64 (row, k) elements they hold.
HC_HD void unpack_lane_words(const uint32_t* words, int lane, int bits, int g, int rb,
                             uint8_t* q /* [N][K] */, int K) {
  for (int j = 0; j < 8; ++j) {
    for (int i = 0; i < 4; ++i) {
      const Slot s = slot(bits, j, i);
      uint32_t reg = 0u;                       // the kernel's register minus the magic bits
      for (int p = 0; p < s.nparts; ++p) {
        const Part& pt = s.p[p];
        uint32_t m = ((1u << pt.nbits) - 1u) << pt.pos;
        m |= m << 16;
        reg |= (words[pt.word] >> pt.shift) & m;
      }
      for (int h = 0; h < 2; ++h) {
        const uint32_t half = (reg >> (16 * h)) & 0xFFFFu;
        const uint32_t qv = (half >> s.fp) & ((1u << bits) - 1u);
        const int row = rb * kRows + frag_row(lane, i);
        const int k = g * kGroup + frag_k(lane, j, i, h);
        q[(size_t)row * K + k] = (uint8_t)qv;
      }
    }
  }
}

}  // namespace hc
