// Device helpers shared by the per-window decode kernel (decode.cu) and the persistent stack kernel
// (stack.cu): async-copy / mbarrier wrappers, the mma.sync tiles and the record (layout.h) decoding.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "decode.h"
#include "layout.h"

namespace hc {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// counter += v with release semantics (orders the writes made before it — by this thread, or by others
// ordered before it through a warp / CTA barrier — without a sequentially consistent fence)
__device__ __forceinline__ unsigned add_release(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// counter += v with acquire-release semantics: the CTA that completes a window (and then resets the
// window's accumulators and counters) also observes every other CTA's released writes
__device__ __forceinline__ unsigned add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// System-scope variants for peer mode (counters incremented by other GPUs over NVLink).
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Bounded spin on a peer counter: a peer that never arrives (crashed rank, mis-set peer table) traps after
// ~20 s instead of hanging the GPU.
__device__ __forceinline__ void wait_sys(const unsigned* p, unsigned target) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_relaxed_sys(p) < target) {
    __nanosleep(64);
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 20000000000ull) __trap();
  }
  (void)ld_acquire_sys(p);
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// W tiles: fp16 A-fragments (1024 + 2^fp·q, exact) times fp16 x' = x·2^-fp
__device__ __forceinline__ void mma16816_f16(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t hf2_sub(uint32_t a, uint32_t b) {
  __half2 r = __hsub2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ float bf16_bits_to_f32(uint32_t h) { return __uint_as_float(h << 16); }
__device__ __forceinline__ uint32_t f32_to_bf16_rn(float f) {
  __nv_bfloat16 b = __float2bfloat16_rn(f);
  return (uint32_t)(*reinterpret_cast<uint16_t*>(&b));
}
// t as a bf16 hi + lo pair per value (fp32-accurate B operand of the U·t mma), two values per register: one packed
// RN conversion per pair (F2FP) instead of two; a in the low half, b in the high half
__device__ __forceinline__ void t_hi_lo(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(a - bf16_bits_to_f32(hi & 0xFFFFu), b - bf16_bits_to_f32(hi >> 16));
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// (a & b) | c in one LOP3 (nvcc otherwise emits two)
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// w >> s; shifts of 8 or more run as IMAD.HI on the FMA pipe to balance it against the ALU pipe
// (which carries the LOP3s)
__device__ __forceinline__ uint32_t shr(uint32_t w, int s) {
  return s == 0 ? w : (s >= 8 ? __umulhi(w, 1u << (32 - s)) : (w >> s));
}

template <int BITS>
__device__ __forceinline__ uint32_t extract(const uint32_t (&w)[2 * BITS], int j, int i) {
  const Slot s = slot(BITS, j, i);
  uint32_t acc = kMagic;
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    if (p < s.nparts) {
      uint32_t m = ((1u << s.p[p].nbits) - 1u) << s.p[p].pos;
      m |= m << 16;
      acc = and_or(shr(w[s.p[p].word], s.p[p].shift), m, acc);
    }
  }
  return acc;
}

// A warp's share of one CTA work item: n tiles at base + t*tb (tb bytes each).
struct Share {
  const uint8_t* base;
  int n, tb, g0, member, is_v;
};

__device__ __forceinline__ int member_of_rb(const DArgs& a, int rb) {
  int m = 0;
#pragma unroll
  for (int i = 1; i < kMaxMembers; ++i)
    if (i < a.n_members && rb >= a.m[i].rb_begin) m = i;
  return m;
}
__device__ __forceinline__ int member_of_chunk(const DArgs& a, int cc) {
  int m = 0;
#pragma unroll
  for (int i = 0; i < kMaxMembers; ++i)
    if (i < a.n_members && a.m[i].r > 0 && cc >= a.m[i].chunk_begin) m = i;
  return m;
}

// The tiles of one row-block item a tile warp streams: contiguous group range [g0, g0 + n).
template <int BITS, int NW = kDecodeWarps>
__device__ __forceinline__ Share warp_share(const DArgs& a, int rb, int warp) {
  Share s;
  s.member = member_of_rb(a, rb);
  const DMember& m = a.m[s.member];
  const int g0 = warp * a.G / NW, g1 = (warp + 1) * a.G / NW;
  s.n = g1 - g0;
  s.g0 = g0;
  s.base = m.rec + ((size_t)(rb - m.rb_begin) * a.G + g0) * rec_bytes(BITS);
  s.tb = rec_bytes(BITS);
  s.is_v = 0;
  return s;
}

// V piece vp of the window (chunk-major, then group, then part p of 2 k16 steps): 1 KB of fragments
__device__ __forceinline__ const uint8_t* v_piece(const DArgs& a, int vp, int& g, int& part) {
  const int per_chunk = 4 * a.G;
  const int cc = vp / per_chunk, rem = vp - cc * per_chunk;
  g = rem >> 2;
  part = rem & 3;
  const DMember& m = a.m[member_of_chunk(a, cc)];
  return reinterpret_cast<const uint8_t*>(m.V + ((size_t)(cc - m.chunk_begin) * a.G * 256 + (size_t)rem * 64));
}

// fp8 (e4m3) factors: V piece vp of a window = (chunk cc, group g, half p2): steps 4·p2 .. 4·p2 + 3 of the
// (chunk, group), 16 ranks x 64 k in 1 KB (repack.cu repack_v8_kernel).
__device__ __forceinline__ const uint8_t* v_piece8(const DArgs& a, int vp, int& g, int& p2) {
  const int per_chunk = 2 * a.G;
  const int cc = vp / per_chunk, rem = vp - cc * per_chunk;
  g = rem >> 1;
  p2 = rem & 1;
  const DMember& m = a.m[member_of_chunk(a, cc)];
  return reinterpret_cast<const uint8_t*>(m.V) + ((size_t)(cc - m.chunk_begin) * a.G * 2 + rem) * 1024;
}

// Two e4m3 bytes (bytes 0 and 1 of w) -> bf16x2, exactly: the byte's magnitude bits placed in a bf16 as
// exponent field e and mantissa m << 4 give value·2^-120 for normals and subnormals alike (a bf16
// subnormal for e = 0), and x 2^120 in bf16 is exact.
__device__ __forceinline__ uint32_t e4m3x2_bf16x2(uint32_t w) {
  const uint32_t t = __byte_perm(w, 0u, 0x4140);                 // byte 0 -> bits 0-7, byte 1 -> bits 16-23
  const uint32_t r = ((t & 0x007F007Fu) << 4) | ((t & 0x00800080u) << 8);
  __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162*>(&r);
  v = __hmul2(v, __floats2bfloat162_rn(0x1p120f, 0x1p120f));
  return *reinterpret_cast<const uint32_t*>(&v);
}
// 8 e4m3 bytes of an A fragment (byte 2i + h = register i, half h) -> the 4 bf16x2 registers.
__device__ __forceinline__ void e4m3x8_frag(const uint2 v, uint32_t (&af)[4]) {
  af[0] = e4m3x2_bf16x2(v.x);
  af[1] = e4m3x2_bf16x2(v.x >> 16);
  af[2] = e4m3x2_bf16x2(v.y);
  af[3] = e4m3x2_bf16x2(v.y >> 16);
}

#ifndef HC_VPW
#define HC_VPW 1
#endif
constexpr int kVPerWarp = HC_VPW;                    // V·x pieces per tile warp of the V CTAs
constexpr float kTScale = 268435456.f;          // 2^28: fixed-point scale of the t accumulators
constexpr float kTInv = 1.f / 268435456.f;

// t accumulators (R22): four tiers of 64-bit integer words, laid out [chunk][tier][16 batch cols][16 ranks]
// (the 16 ranks of one (chunk, tier, col) are one 128-byte line) + one "extra tiers used" flag word after
// the last chunk.  A fp32 partial v goes to exactly ONE tier, chosen by magnitude:
//   tier 0: 2^-24 <= |v| < 2^12  in 2^-36 fixed point   (the common case: the only tier read and reset)
//   tier 1: |v| >= 2^12          in 2^-12 fixed point   (outlier activations; saturates at 2^50)
//   tier 2: 2^-48 <= |v| < 2^-24 in 2^-72 fixed point   (tiny activations)
//   tier 3: |v| < 2^-48          in 2^-96 fixed point
// Each partial is rounded once with |error| <= 2^-25·max(|v|, 2^-24·2^-12) in tier 0 and relative error
// <= 2^-25 (one fp32 rounding) in tiers 1-3 (tier 3: down to |v| = 2^-72); a tier stays below 2^48 per
// partial, 2^63 for up to 2^15 partials.  The tier-0 band is wide so that partials of ordinary activations
// (including the occasional near-cancelled one: a normal partial falls below 2^-24 with probability
// ~1e-6) never leave it; whole windows of tiny or huge activations set the flag.  Integer adds are
// order-free: t is deterministic.  One atomic per partial; the common case reads and resets one word per
// element.
// Predicated L2 load (no branch: the predicate goes on the load, so a batch of these stays one round trip).
__device__ __forceinline__ long long ldcg_if(const long long* p, bool on) {
  long long v;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b64 %0, 0;\n @q ld.global.cg.b64 %0, [%1];\n}"
               : "=l"(v) : "l"(p), "r"((int)on) : "memory");
  return v;
}
__device__ __forceinline__ size_t tacc_idx(int cc, int w, int rank, int col) {
  return (size_t)cc * kTChunk + (w * 16 + col) * 16 + rank;
}
__device__ __forceinline__ void tacc_add(long long* t, int n_chunks, int cc, int col, int rank, float v) {
  const float a = fabsf(v);
  const int w = a >= 0x1p-24f ? (a >= 0x1p12f ? 1 : 0) : (a >= 0x1p-48f ? 2 : 3);
  const int se = w == 0 ? 36 : (w == 1 ? 12 : (w == 2 ? 72 : 96));
  const float q = fminf(fmaxf(v * __uint_as_float((uint32_t)(127 + se) << 23), -0x1p62f), 0x1p62f);   // exact scaling
  const long long iq = __float2ll_rn(q);
  if (iq != 0) {
    const size_t cp = (size_t)(blockIdx.x % kTCopies) * n_chunks * kTChunk;   // this CTA's copy
    atomicAdd(reinterpret_cast<unsigned long long*>(t + cp + tacc_idx(cc, w, rank, col)), (unsigned long long)iq);
    if (w != 0) t[(size_t)kTCopies * n_chunks * kTChunk] = 1;   // extra tiers in use (idempotent plain store)
  }
}
// 0, computed from v by an opaque instruction: a data dependency on v that the compiler cannot fold
__device__ __forceinline__ unsigned zero_dep(unsigned v) {
  unsigned z;
  asm("and.b32 %0, %1, 0;" : "=r"(z) : "r"(v));
  return z;
}
// Predicated L2 load without a compiler barrier (the deep t pass: loads of several elements stay in flight together;
// the data was ordered by the caller's acquire)
__device__ __forceinline__ long long ldcg_if_nb(const long long* p, bool on) {
  long long v;
  asm("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n mov.b64 %0, 0;\n @q ld.global.cg.b64 %0, [%1];\n}"
      : "=l"(v) : "l"(p), "r"((int)on));
  return v;
}
// Extra-tier t pass (R22: the window's flag is set, outlier or tiny activations): the t fragments of the epilogue's
// U·t mma are rebuilt from all four tiers.  Load: the 32 lanes convert distinct (chunk, live column, rank) elements
// into fp32 scratch laid over the chunk's own fragment slots ([cc][col < 8·NB8][rank], exactly NB8 x 512 B), every
// load in flight together (one L2 round trip for any chunk count); per element t = t0·2^-36 + (t1·2^-12 +
// (t2·2^-72 + t3·2^-96)) in fp32.  Build (t_fragments_build), chunk by chunk: each lane reads its four values per
// batch-column block, then the chunk's slots are overwritten with the fragments (ranks >= r masked; fp8 factors:
// t'_j = u_scale_j·t_j).  tq = the accumulators, carrying a data dependency on the acquire (the loads are
// non-volatile so that they batch).
template <int NB8>
__device__ __forceinline__ void t_fragments_deep_load(const DArgs& a, const long long* tq, uint4* tsm, int lane) {
  constexpr int kCol = 8 * NB8;
  static_assert(kTCopies == 1, "extra-tier pass: one accumulator copy");
  float* scr = reinterpret_cast<float*>(tsm);
  __syncwarp();                                          // the tier-0 fragments are overwritten below
  const int per = a.B * 16, n_el = a.n_chunks * per;     // only the B live columns (build reads zero for the others)
#pragma unroll 4
  for (int e = lane; e < n_el; e += 32) {
    const int cc = e / per, rem = e - cc * per;          // rem = col · 16 + rank
    const long long* p = tq + (size_t)cc * kTChunk + rem;
    scr[cc * kCol * 16 + rem] = (float)ldcg_if_nb(p, true) * 0x1p-36f +
                                fmaf((float)ldcg_if_nb(p + 256, true), 0x1p-12f,
                                     fmaf((float)ldcg_if_nb(p + 512, true), 0x1p-72f,
                                          (float)ldcg_if_nb(p + 768, true) * 0x1p-96f));
  }
  __syncwarp();
}
template <int NB8>
__device__ __forceinline__ void t_fragments_build(const DArgs& a, uint4* tsm, int lane) {
  const int gid = lane >> 2, tig = lane & 3;
  constexpr int kCol = 8 * NB8;
  const float* scr = reinterpret_cast<const float*>(tsm);
  for (int cc = 0; cc < a.n_chunks; ++cc) {
    const DMember& mt = a.m[member_of_chunk(a, cc)];
    const int r0 = 16 * (cc - mt.chunk_begin) + 2 * tig;
    float tr[NB8][4];
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb) {
      const float* src = scr + (size_t)cc * kCol * 16 + (gid + 8 * nb) * 16 + 2 * tig;
      const bool on = gid + 8 * nb < a.B;
      tr[nb][0] = on ? src[0] : 0.f; tr[nb][1] = on ? src[1] : 0.f; tr[nb][2] = on ? src[8] : 0.f; tr[nb][3] = on ? src[9] : 0.f;
    }
    __syncwarp();
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb) {
      uint32_t hi[2], lo[2];
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int ra = r0 + 8 * hh, rb = ra + 1;
        float ta = ra < mt.r ? tr[nb][2 * hh] : 0.f;
        float tb = rb < mt.r ? tr[nb][2 * hh + 1] : 0.f;
        if (a.fp8) {
          ta *= ra < mt.r ? mt.us[ra] : 0.f;
          tb *= rb < mt.r ? mt.us[rb] : 0.f;
        }
        t_hi_lo(ta, tb, hi[hh], lo[hh]);
      }
      tsm[((size_t)cc * NB8 + nb) * 32 + lane] = make_uint4(hi[0], hi[1], lo[0], lo[1]);
    }
    __syncwarp();
  }
}
// Reset what a launch with batch B wrote: tier 0 always, tiers 1-3 and the flag when `xt` (the flag as the
// caller read it; plain stores only on this exit path, no load); one warp.
__device__ __forceinline__ void tacc_reset(long long* t, int n_chunks, int B, bool xt, int lane) {
  const int per = B * 16, tiers = xt ? kTTiers : 1;      // words of one (copy, chunk, tier): cols < B x 16 ranks
  for (int i = lane; i < kTCopies * n_chunks * tiers * per; i += 32) {
    const int row = i / per;                             // (copy · n_chunks + chunk) · tiers + tier
    const int c = row / tiers, w = row - c * tiers;
    const int j = i - row * per;                         // col · 16 + rank
    t[(size_t)c * kTChunk + tacc_idx(0, w, j & 15, j >> 4)] = 0;
  }
  if (lane == 0 && xt) t[(size_t)kTCopies * n_chunks * kTChunk] = 0;
}

// Row of x used by mma column `col` (batch index).  Columns >= B read a valid row; their
// outputs are never stored, so no zeroing is needed.
__device__ __forceinline__ int xrow(const DArgs& a, int col) { return col < a.B ? col : a.B - 1; }

// ---- per-(group, batch row) power-of-two prescale of the fp16 B operand (R20).
// x' = x·2^-(fp + σ) (fp <= 4 for the B operand) is exact in fp16 for every bf16 x with |x|·2^-(fp+σ) in
// [2^-17, 2^15] (fp16's 11-bit significand holds bf16's 8 bits down to the subnormal grid 2^-24).
// σ = 0 whenever the group's largest |x| has exponent E in [-6, 13] (the common case: no extra work,
// bit-identical to no prescale): x' < 2^14, and an element below 2^-13 rounds to the fp16 subnormal grid
// with |error| <= 2^-21 <= 2^-15·max|x| of its group (a bounded, not an exact, product — R20).
// Otherwise σ = E - 12 (the group's largest |x'| lands in [2^12, 2^13)), clamped to [-100, 115] so that
// 2^±σ stay normal floats: elements within 2^-29 of the group max are exact, smaller ones round with
// |error| <= 2^-42·max.  The group's fp32 partial sum is multiplied back by 2^σ (exact: a power of two).
// So the full bf16 range is accepted: outliers >= 65504 and tiny (< 2^-14) activations included.
// Zero and non-finite groups keep σ = 0 (inf / NaN propagate through the products).
__device__ __forceinline__ int prescale_sigma(uint32_t m) {   // m = the group's largest |x| (bf16 bits & 0x7FFF)
  if (m == 0 || m >= 0x7F80u) return 0;
  const int E = max((int)(m >> 7), 1) - 127;
  if (E >= -6 && E <= 13) return 0;
  return min(max(E - 12, -100), 115);
}
__device__ __forceinline__ float pow2i(int e) { return __uint_as_float((uint32_t)(127 + e) << 23); }   // e in [-126, 127]

// x' fragments of group g from the window's fp16 x' buffer (global, L1-cached):
// xr[nb][4q + e] = x'[b][g*128 + 32q + 8tig .. +7]
// NC: read-only path (x' written before the launch); !NC: coherent weak loads, for x' written by an
// earlier window of the same launch (persistent stack kernel; ordered by an acquire + bar.sync)
template <int NB8, bool NC = true>
__device__ __forceinline__ void load_x_global(const DArgs& a, int g, int lane, uint32_t (&xr)[NB8][16]) {
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb) {
    const uint4* p = reinterpret_cast<const uint4*>(a.x16 + (size_t)xrow(a, (lane >> 2) + 8 * nb) * a.K +
                                                    g * kGroup + 8 * (lane & 3));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint4 v;
      if (NC) v = __ldg(p + 4 * q);
      else asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + 4 * q));
      xr[nb][4 * q + 0] = v.x; xr[nb][4 * q + 1] = v.y; xr[nb][4 * q + 2] = v.z; xr[nb][4 * q + 3] = v.w;
    }
  }
}

// Largest |x| (bf16 bits without the sign) of the 8 bf16 values in a uint4.
__device__ __forceinline__ uint32_t absmax8(const uint4 v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) m = max(m, max(w[i] & 0x7FFFu, (w[i] >> 16) & 0x7FFFu));
  return m;
}

// Slow path of the x' hand-off (stack windows whose producer flagged an x' value fp16 cannot hold
// exactly, R20): read bf16 x of group g from global memory, take the per-(group, column)
// prescale from the group's largest |x| (the four tig lanes of a column hold its 128 k), and build the
// same fragments as load_x_global plus the output-column factors fs.
template <int BITS, int NB8>
__device__ __forceinline__ void load_x_bf16_sig(const DArgs& a, int g, int lane, uint32_t (&xr)[NB8][16],
                                                float (&fs)[NB8][2]) {
  const int gid = lane >> 2, tig = lane & 3;
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb) {
    const uint4* p = reinterpret_cast<const uint4*>(a.x + (size_t)xrow(a, gid + 8 * nb) * a.ldx + g * kGroup + 8 * tig);
    uint4 v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = __ldcg(p + 4 * q);          // k = 32q + 8tig .. +7
    uint32_t m = max(max(absmax8(v[0]), absmax8(v[1])), max(absmax8(v[2]), absmax8(v[3])));
    m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, 1));
    m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, 2));
    const int sig = prescale_sigma(m);                             // column gid + 8nb, group g
    const float ps = pow2i(-sig);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t wv[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
#pragma unroll
      for (int w2 = 0; w2 < 4; ++w2) {                             // k pair 32q + 8tig + 2w2 (+1)
        const float c = __uint_as_float((uint32_t)(127 - step_fp(BITS, 2 * q + ((w2 >> 1) & 1), w2 & 1)) << 23);
        const __half2 hv = __floats2half2_rn((bf16_bits_to_f32(wv[w2] & 0xFFFFu) * c) * ps,
                                             (bf16_bits_to_f32(wv[w2] >> 16) * c) * ps);
        xr[nb][4 * q + w2] = *reinterpret_cast<const uint32_t*>(&hv);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) fs[nb][h] = pow2i(__shfl_sync(0xFFFFFFFFu, sig, (2 * tig + h) * 4));
  }
}

// One (row-block, group) record: tot[nb][e] += s_row · Σ_k (q − z)·x.
// The A registers hold 2^fp·(q − z) (fp16, exact) and the B operand is x' = x·2^-fp (fp16), so every
// product is exact and one mma chain accumulates Σ_k (q − z)·x_k in fp32.
// XS: x' fragments come from shared memory (xrow_s[nb] = this lane's run start for the group).
// The compute part of w_tile on a record already in registers (w = the lane's code words, sw = its
// scales word, zz = the record's zeros).
// SIG: the B operand carries a per-(group, column) prescale 2^-σ; fs[nb][h] = 2^σ of output column
// 2·tig + h + 8·nb multiplies the group's partial back (exact).
template <int BITS, int NB8, bool XS, bool SIG = false>
__device__ __forceinline__ void w_tile_regs(const uint32_t (&w)[2 * BITS], uint32_t sw, uint2 zz, int lane,
                                            const uint4* const (&xrow_s)[NB8], const uint32_t (&xr)[NB8][16],
                                            float (&tot)[NB8][4], const float (&fs)[NB8][2]) {
  const int gid = lane >> 2;
  // fp16x2 (1024 + 2^fp·z) of rows gid / gid + 8 for each field exponent fp: subtracting it turns a
  // register into 2^fp·(q − z) exactly, so the mma accumulates Σ (q − z)·x with no large offset
  const uint32_t zr0 = (zz.x >> (4 * gid)) & 15u, zr1 = (zz.y >> (4 * gid)) & 15u;
  auto zc = [&](int row_hi, int fp) -> uint32_t { return (0x6400u + ((row_hi ? zr1 : zr0) << fp)) * 0x00010001u; };
  float acc[NB8][4];
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nb][e] = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t xq[NB8][4];
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb) {
      if constexpr (XS) {
        const uint4 v = xrow_s[nb][4 * q];
        xq[nb][0] = v.x; xq[nb][1] = v.y; xq[nb][2] = v.z; xq[nb][3] = v.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) xq[nb][e] = xr[nb][4 * q + e];
      }
    }
#pragma unroll
    for (int jj = 0; jj < 2; ++jj) {
      const int j = 2 * q + jj;
      uint32_t af[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        af[i] = extract<BITS>(w, j, i);                            // 1024 + 2^fp·q (exact)
        af[i] = hf2_sub(af[i], zc(i & 1, slot(BITS, j, i).fp));   // 2^fp·(q − z) (exact)
      }
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb) mma16816_f16(acc[nb], af, xq[nb][2 * jj], xq[nb][2 * jj + 1]);
    }
  }
  // row gid + 8 registers may carry 2^row_hi_shift (layout.h): exact power-of-two rescale
  const float s0 = bf16_bits_to_f32(sw & 0xFFFFu),
              s1 = bf16_bits_to_f32(sw >> 16) * (1.f / (float)(1 << row_hi_shift(BITS)));
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb) {
    if constexpr (SIG) {
      tot[nb][0] = fmaf(s0 * fs[nb][0], acc[nb][0], tot[nb][0]);
      tot[nb][1] = fmaf(s0 * fs[nb][1], acc[nb][1], tot[nb][1]);
      tot[nb][2] = fmaf(s1 * fs[nb][0], acc[nb][2], tot[nb][2]);
      tot[nb][3] = fmaf(s1 * fs[nb][1], acc[nb][3], tot[nb][3]);
    } else {
      tot[nb][0] = fmaf(s0, acc[nb][0], tot[nb][0]);
      tot[nb][1] = fmaf(s0, acc[nb][1], tot[nb][1]);
      tot[nb][2] = fmaf(s1, acc[nb][2], tot[nb][2]);
      tot[nb][3] = fmaf(s1, acc[nb][3], tot[nb][3]);
    }
  }
}

template <int BITS, int NB8, bool XS, bool SIG = false>
__device__ __forceinline__ void w_tile(const uint8_t* rec, int lane, const uint4* const (&xrow_s)[NB8],
                                       const uint32_t (&xr)[NB8][16], float (&tot)[NB8][4], const float (&fs)[NB8][2]) {
  uint32_t w[2 * BITS];
#pragma unroll
  for (int q = 0; q < (2 * BITS) / 4; ++q) {
    const uint4 v = *reinterpret_cast<const uint4*>(rec + q * 512 + lane * 16);
    w[4 * q + 0] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
  }
  if constexpr ((2 * BITS) % 4) {
    const uint2 v = *reinterpret_cast<const uint2*>(rec + 512 * ((2 * BITS) / 4) + lane * 8);
    w[2 * BITS - 2] = v.x; w[2 * BITS - 1] = v.y;
  }
  const int gid = lane >> 2;
  const uint32_t sw = *reinterpret_cast<const uint32_t*>(rec + scales_off(BITS) + 4 * gid);
  const uint2 zz = *reinterpret_cast<const uint2*>(rec + zeros_off(BITS));   // rows 0..7 | rows 8..15
  w_tile_regs<BITS, NB8, XS, SIG>(w, sw, zz, lane, xrow_s, xr, tot, fs);
}

// Load the lane's part of one record (code words, scales word, zeros) from shared or global memory.
template <int BITS>
__device__ __forceinline__ void load_record(const uint8_t* rec, int lane, uint32_t (&w)[2 * BITS], uint32_t& sw,
                                            uint2& zz) {
#pragma unroll
  for (int q = 0; q < (2 * BITS) / 4; ++q) {
    const uint4 v = *reinterpret_cast<const uint4*>(rec + q * 512 + lane * 16);
    w[4 * q + 0] = v.x; w[4 * q + 1] = v.y; w[4 * q + 2] = v.z; w[4 * q + 3] = v.w;
  }
  if constexpr ((2 * BITS) % 4) {
    const uint2 v = *reinterpret_cast<const uint2*>(rec + 512 * ((2 * BITS) / 4) + lane * 8);
    w[2 * BITS - 2] = v.x; w[2 * BITS - 1] = v.y;
  }
  sw = *reinterpret_cast<const uint32_t*>(rec + scales_off(BITS) + 4 * (lane >> 2));
  zz = *reinterpret_cast<const uint2*>(rec + zeros_off(BITS));
}

// x' = x·2^-fp (fp16) of 16 consecutive k of one batch row: `part` (0..7) selects k = 16·part .. +15
// within the group; fp is the code-field exponent of that k's column pair (layout.h).  Shared by the
// in-kernel staging pass (XS) and the x-prep kernel (global x').
template <int BITS>
__device__ __forceinline__ void xprime16(const uint4 (&in)[2], int part, uint4 (&out)[2], int sig = 0) {
  const float ps = pow2i(-sig);                                        // the group's prescale 2^-σ
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t wv[4] = {in[h].x, in[h].y, in[h].z, in[h].w};
    uint32_t ov[4];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      float xp[2];
#pragma unroll
      for (int hi = 0; hi < 2; ++hi) {
        const int k = part * 16 + h * 8 + 2 * e2 + hi;               // k within the group
        const int j = 2 * (k >> 5) + ((k >> 2) & 1), pr = (k >> 1) & 1;
        const float xv = bf16_bits_to_f32((wv[e2] >> (16 * hi)) & 0xFFFFu);
        xp[hi] = (xv * __uint_as_float((uint32_t)(127 - step_fp(BITS, j, pr)) << 23)) * ps;
      }
      const __half2 hv = __floats2half2_rn(xp[0], xp[1]);
      ov[e2] = *reinterpret_cast<const uint32_t*>(&hv);
    }
    out[h] = make_uint4(ov[0], ov[1], ov[2], ov[3]);
  }
}

// One 1 KB V piece = steps 2p, 2p+1 of a (chunk, group) tile; xv = the lane's 16 B x run.
template <int NB8>
__device__ __forceinline__ void v_tile(const uint8_t* piece, int lane, const uint4 (&xv)[NB8], float (&tot)[NB8][4]) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const uint4 v = *reinterpret_cast<const uint4*>(piece + s * 512 + lane * 16);
    const uint32_t af[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb) {
      if (s == 0) mma16816(tot[nb], af, xv[nb].x, xv[nb].y);
      else        mma16816(tot[nb], af, xv[nb].z, xv[nb].w);
    }
  }
}

// fp8 V piece (4 steps, 16 ranks x 64 k): xa / xb = the lane's x runs of the piece's two 32-k halves.
template <int NB8>
__device__ __forceinline__ void v_tile8(const uint8_t* piece, int lane, const uint4 (&xa)[NB8], const uint4 (&xb)[NB8],
                                        float (&tot)[NB8][4]) {
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    uint32_t af[4];
    e4m3x8_frag(*reinterpret_cast<const uint2*>(piece + s * 256 + lane * 8), af);
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb) {
      const uint4& xx = s < 2 ? xa[nb] : xb[nb];
      mma16816(tot[nb], af, (s & 1) ? xx.z : xx.x, (s & 1) ? xx.w : xx.y);
    }
  }
}

// The next window's x' (fp16, pre-scaled by the code-field exponent of its column pair, layout.h) of
// one output element (bf16 bits) at output column n, batch row b.  Values outside the σ = 0 band of
// their group are fixed up by the consumer (x16_max, R20).
template <int BITS>
__device__ __forceinline__ void write_xprime(const DArgs& a, int b, int n, uint16_t bits) {
  const int k = n - a.y16_lo, kk = k & (kGroup - 1);
  const int j = 2 * (kk >> 5) + ((kk >> 2) & 1), pr = (kk >> 1) & 1;
  const int fp = step_fp(BITS, j, pr);
  const float xv = bf16_bits_to_f32(bits) * __uint_as_float((uint32_t)(127 - fp) << 23);
  a.y16[(size_t)b * (a.y16_hi - a.y16_lo) + k] = __half_as_ushort(__float2half_rn(xv));
}

// Publish the largest |x| of this lane's hand-off values per batch row into y16_max[g][b] (g = the next
// window's group of output column n0).  m[nb][h] = the lane's max for batch row 2tig + h + 8nb; the
// 8 gid lanes of a tig are reduced first, then one atomicMax per (group, batch row).
template <int NB8>
__device__ __forceinline__ void publish_xmax(const DArgs& a, int n0, const uint32_t (&m)[NB8][2], int lane) {
  const int g = (n0 - a.y16_lo) >> 7, tig = lane & 3;
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t v = m[nb][h];
      v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, 4));
      v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, 8));
      v = max(v, __shfl_xor_sync(0xFFFFFFFFu, v, 16));
      const int b = 2 * tig + h + 8 * nb;
      if ((lane >> 2) == 0 && b < a.B && v != 0) atomicMax(a.y16_max + g * 16 + b, v);
    }
}

}  // namespace

}  // namespace hc
