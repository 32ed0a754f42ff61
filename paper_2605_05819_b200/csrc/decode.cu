// Fused decode kernel: one launch evaluates a whole compensation window
//
//     y[b, n] = Σ_g s[n,g] · Σ_{k∈g} (q[n,k] − z[n,g]) · x[b,k]  +  Σ_{j<r} U[n,j] · t[b,j],
//     t[b, j] = Σ_k V[j,k] · x[b,k]                                      (north_star)
//
// Design (DESIGN.md §"Decode kernel"):
//  * persistent grid, 8 warps per CTA; CTA work items are (a) rank-projection items
//    (16 ranks × a K-slice of V) and then (b) row-block items (16 output rows × all K);
//  * each warp streams its tiles (one (row-block, group) record or one 1 KB V piece) from
//    HBM with cp.async.bulk (TMA engine) into a private 4-slot shared-memory ring guarded by
//    mbarriers, L2 evict-first; W is never materialised;
//  * codes -> bf16 A-fragments with shift/lop3 and the 0x4300 magic (exact integers), minus
//    the per-group zero (exact), contracted with bf16 x on mma.sync m16n8k16 (fp32 accumulate),
//    per-group partial sums scaled by the fp32 group scale afterwards (no bf16 rounding of W);
//  * the 8 warps' partial sums are reduced in shared memory; the CTA's epilogue warp adds
//    U[:, :r]·t with t split into bf16 hi + lo (fp32-accurate) on the same mma, then writes y
//    once (fp32, or bf16 = RNE of the fp32 value), optionally adding a bf16 residual;
//  * t is produced inside the same launch: rank-projection items publish per-slice partials,
//    the last arriver per chunk reduces them in a fixed order (deterministic) and bumps a
//    release counter that row-block epilogues acquire.  Counters self-reset at the end.
#include <cuda_bf16.h>
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

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t bf2_sub(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hsub2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t bf2_mul(uint32_t a, uint32_t b) {
  __nv_bfloat162 r = __hmul2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
  return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ float bf16_bits_to_f32(uint32_t h) { return __uint_as_float(h << 16); }
__device__ __forceinline__ uint32_t f32_to_bf16_rn(float f) {
  __nv_bfloat16 b = __float2bfloat16_rn(f);
  return (uint32_t)(*reinterpret_cast<uint16_t*>(&b));
}

// 2^-fp as a bf16x2 constant
__device__ __forceinline__ constexpr uint32_t pow2neg_bf16x2(int fp) {
  return (uint32_t)(0x3F80 - (fp << 7)) * 0x00010001u;
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
      acc |= (w[s.p[p].word] >> s.p[p].shift) & m;
    }
  }
  return acc;
}

struct Tiles {   // a warp's share of one CTA work item
  int n;         // number of tiles
  int g0;        // first group
};

__device__ __forceinline__ Tiles warp_tiles(const DArgs& a, int item, int warp) {
  const int nV = a.n_chunks * a.vks;
  if (item < nV) {
    const int vs = item % a.vks;
    const int lo = vs * a.G / a.vks, hi = (vs + 1) * a.G / a.vks;
    const int g0 = lo + warp * (hi - lo) / kDecodeWarps, g1 = lo + (warp + 1) * (hi - lo) / kDecodeWarps;
    return Tiles{4 * (g1 - g0), g0};
  }
  const int g0 = warp * a.G / kDecodeWarps, g1 = (warp + 1) * a.G / kDecodeWarps;
  return Tiles{g1 - g0, g0};
}

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

template <int BITS>
__device__ __forceinline__ const void* tile_src(const DArgs& a, int item, int g0, int t, uint32_t& bytes) {
  const int nV = a.n_chunks * a.vks;
  if (item < nV) {
    const int cc = item / a.vks;
    const DMember& m = a.m[member_of_chunk(a, cc)];
    const int c = cc - m.chunk_begin, g = g0 + (t >> 2), p = t & 3;
    bytes = 1024;
    return m.V + ((size_t)(c * a.G + g) * 8 + 2 * p) * 32;
  }
  const int rb = item - nV;
  const DMember& m = a.m[member_of_rb(a, rb)];
  bytes = rec_bytes(BITS);
  return m.rec + ((size_t)(rb - m.rb_begin) * a.G + (g0 + t)) * rec_bytes(BITS);
}

// x fragments of group g for the lane: xr[nb][16] (bf16x2), step j uses xr[nb][2j], xr[nb][2j+1]
template <int NB8>
__device__ __forceinline__ void load_x(const DArgs& a, int g, int lane, uint32_t (&xr)[NB8][16]) {
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb) {
    const int b = (lane >> 2) + 8 * nb;
    if (b < a.B) {
      const uint4* p = reinterpret_cast<const uint4*>(a.x + (size_t)b * a.K + g * kGroup + 32 * (lane & 3));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = __ldg(p + q);
        xr[nb][4 * q + 0] = v.x; xr[nb][4 * q + 1] = v.y; xr[nb][4 * q + 2] = v.z; xr[nb][4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) xr[nb][q] = 0u;
    }
  }
}

// One (row-block, group) record: tot[nb][e] += s_row · Σ_k (q − z)·x
template <int BITS, int NB8>
__device__ __forceinline__ void w_tile(const uint8_t* rec, int lane, const uint32_t (&xr)[NB8][16],
                                       float (&tot)[NB8][4]) {
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
  const uint64_t zw = *reinterpret_cast<const uint64_t*>(rec + zeros_off(BITS));
  const float s0 = bf16_bits_to_f32(sw & 0xFFFFu), s1 = bf16_bits_to_f32(sw >> 16);
  const uint32_t z[2] = {(uint32_t)(zw >> (4 * gid)) & 15u, (uint32_t)(zw >> (4 * gid + 32)) & 15u};
  float acc[NB8][4];
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nb][e] = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    uint32_t af[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int fp = slot(BITS, j, i).fp;
      const uint32_t zc = (0x4300u + (z[i & 1] << fp)) * 0x00010001u;   // bf16x2(128 + z·2^fp), exact
      af[i] = bf2_sub(extract<BITS>(w, j, i), zc);                       // 2^fp·(q − z), exact
    }
    const int fp0 = step_fp(BITS, j, 0), fp1 = step_fp(BITS, j, 1);
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb) {
      uint32_t b0 = xr[nb][2 * j], b1 = xr[nb][2 * j + 1];
      if (fp0) b0 = bf2_mul(b0, pow2neg_bf16x2(fp0));
      if (fp1) b1 = bf2_mul(b1, pow2neg_bf16x2(fp1));
      mma16816(acc[nb], af, b0, b1);
    }
  }
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb) {
    tot[nb][0] = fmaf(s0, acc[nb][0], tot[nb][0]);
    tot[nb][1] = fmaf(s0, acc[nb][1], tot[nb][1]);
    tot[nb][2] = fmaf(s1, acc[nb][2], tot[nb][2]);
    tot[nb][3] = fmaf(s1, acc[nb][3], tot[nb][3]);
  }
}

// One 1 KB V piece = steps 2p, 2p+1 of a (chunk, group) tile
template <int NB8>
__device__ __forceinline__ void v_tile(const uint8_t* piece, int p, int lane, const uint32_t (&xr)[NB8][16],
                                       float (&tot)[NB8][4]) {
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const uint4 v = *reinterpret_cast<const uint4*>(piece + s * 512 + lane * 16);
    const uint32_t af[4] = {v.x, v.y, v.z, v.w};
    const int j = 2 * p + s;
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb) {
      // j is not a compile-time constant here (p is runtime): index the pair explicitly
      uint32_t b0, b1;
      switch (j) {
        case 0: b0 = xr[nb][0]; b1 = xr[nb][1]; break;
        case 1: b0 = xr[nb][2]; b1 = xr[nb][3]; break;
        case 2: b0 = xr[nb][4]; b1 = xr[nb][5]; break;
        case 3: b0 = xr[nb][6]; b1 = xr[nb][7]; break;
        case 4: b0 = xr[nb][8]; b1 = xr[nb][9]; break;
        case 5: b0 = xr[nb][10]; b1 = xr[nb][11]; break;
        case 6: b0 = xr[nb][12]; b1 = xr[nb][13]; break;
        default: b0 = xr[nb][14]; b1 = xr[nb][15]; break;
      }
      mma16816(tot[nb], af, b0, b1);
    }
  }
}

}  // namespace

template <int BITS, int NB8>
__global__ void __launch_bounds__(kDecodeWarps * 32) decode_kernel(const __grid_constant__ DArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = smem + (size_t)warp * kRing * kSlotBytes;
  float* red = reinterpret_cast<float*>(smem + (size_t)kDecodeWarps * kRing * kSlotBytes);   // [2][8][32][8]
  uint64_t* bars = reinterpret_cast<uint64_t*>(red + 2 * kDecodeWarps * 32 * 8) + warp * kRing;

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < kRing; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  const uint64_t policy = evict_first_policy();

  const int nV = a.n_chunks * a.vks;
  const int n_items = nV + a.n_rb;

  // producer cursor (tiles issued) — warp-uniform state, lane 0 issues
  int p_item = blockIdx.x, p_t = 0;
  Tiles p_tl = p_item < n_items ? warp_tiles(a, p_item, warp) : Tiles{0, 0};
  unsigned issued = 0, consumed = 0;
  auto issue = [&]() {
    while (issued - consumed < (unsigned)kRing && p_item < n_items) {
      if (p_t < p_tl.n) {
        uint32_t bytes;
        const void* src = tile_src<BITS>(a, p_item, p_tl.g0, p_t, bytes);
        const int s = issued % kRing;
        if (lane == 0) bulk_load(ring + s * kSlotBytes, src, bytes, &bars[s], policy);
        ++issued;
        ++p_t;
      } else {
        p_item += gridDim.x;
        p_t = 0;
        p_tl = p_item < n_items ? warp_tiles(a, p_item, warp) : Tiles{0, 0};
      }
    }
  };
  issue();

  int parity = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, parity ^= 1) {
    const Tiles tl = warp_tiles(a, item, warp);
    const bool is_v = item < nV;
    float tot[NB8][4];
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) tot[nb][e] = 0.f;
    uint32_t xr[NB8][16];
    int xg = -1;
    for (int t = 0; t < tl.n; ++t) {
      const int s = consumed % kRing;
      const uint32_t ph = (consumed / kRing) & 1u;
      const int g = is_v ? tl.g0 + (t >> 2) : tl.g0 + t;
      if (g != xg) { load_x<NB8>(a, g, lane, xr); xg = g; }
      while (!mbar_try_wait(&bars[s], ph)) {}
      if (is_v) v_tile<NB8>(ring + s * kSlotBytes, t & 3, lane, xr, tot);
      else      w_tile<BITS, NB8>(ring + s * kSlotBytes, lane, xr, tot);
      __syncwarp();
      ++consumed;
      issue();
    }
    // ---- CTA reduction of the 8 warps' partial sums (fixed order)
    float* rb_ = red + ((size_t)(parity * kDecodeWarps + warp) * 32 + lane) * 8;
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
      *reinterpret_cast<float4*>(rb_ + 4 * nb) = make_float4(tot[nb][0], tot[nb][1], tot[nb][2], tot[nb][3]);
    asm volatile("bar.sync 1, %0;" ::"n"(kDecodeWarps * 32) : "memory");
    if (warp != 0) continue;

    float fin[NB8][4];
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) fin[nb][e] = 0.f;
    for (int w = 0; w < kDecodeWarps; ++w) {
      const float* src = red + ((size_t)(parity * kDecodeWarps + w) * 32 + lane) * 8;
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb) {
        const float4 v = *reinterpret_cast<const float4*>(src + 4 * nb);
        fin[nb][0] += v.x; fin[nb][1] += v.y; fin[nb][2] += v.z; fin[nb][3] += v.w;
      }
    }
    const int gid = lane >> 2, tig = lane & 3;
    if (is_v) {
      // ---- rank projection partial -> last arriver per chunk reduces in slice order
      const int cc = item / a.vks;
      float* vp = a.vpart + ((size_t)item * 32 + lane) * 8;
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
        *reinterpret_cast<float4*>(vp + 4 * nb) = make_float4(fin[nb][0], fin[nb][1], fin[nb][2], fin[nb][3]);
      __threadfence();
      __syncwarp();
      unsigned old = 0;
      if (lane == 0) old = atomicAdd(&a.cnt[cc], 1u);
      old = __shfl_sync(0xffffffffu, old, 0);
      if (old == (unsigned)a.vks - 1) {
        __threadfence();
        float sum[NB8][4];
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) sum[nb][e] = 0.f;
        for (int vs = 0; vs < a.vks; ++vs) {
          const float* src = a.vpart + ((size_t)(cc * a.vks + vs) * 32 + lane) * 8;
#pragma unroll
          for (int nb = 0; nb < NB8; ++nb) {
            const float4 v = __ldcg(reinterpret_cast<const float4*>(src + 4 * nb));
            sum[nb][0] += v.x; sum[nb][1] += v.y; sum[nb][2] += v.z; sum[nb][3] += v.w;
          }
        }
        // fragment: rows = ranks (gid, gid+8), cols = batch (2tig, 2tig+1) + 8nb;  t[cc][b][rank]
        float* tc = a.t + (size_t)cc * 256;
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) tc[(2 * tig + (e & 1) + 8 * nb) * 16 + gid + 8 * (e >> 1)] = sum[nb][e];
        __threadfence();
        __syncwarp();
        if (lane == 0) {
          a.cnt[cc] = 0u;                       // self-reset for the next launch
          atomicAdd(&a.cnt[a.n_chunks], 1u);    // t_done (release via the fence above)
        }
      }
      continue;
    }
    // ---- row-block epilogue: + U[:, :r]·t, residual, output
    const int rb = item - nV;
    const DMember& m = a.m[member_of_rb(a, rb)];
    const int rbl = rb - m.rb_begin;
    float comp[NB8][4];
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) comp[nb][e] = 0.f;
    if (m.r > 0) {
      if (lane == 0)
        while (ld_acquire(&a.cnt[a.n_chunks]) < (unsigned)a.n_chunks) __nanosleep(64);
      __syncwarp();
      const int nck = (m.r + 15) >> 4;
      for (int c = 0; c < nck; ++c) {
        const uint4 u = __ldg(m.U + ((size_t)rbl * (m.r_stored >> 4) + c) * 32 + lane);
        const uint32_t af[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb) {
          const int b = gid + 8 * nb;
          const float* tp = a.t + ((size_t)(m.chunk_begin + c) * 16 + b) * 16;
          float tv[4];
          const float2 v01 = __ldcg(reinterpret_cast<const float2*>(tp + 2 * tig));
          const float2 v89 = __ldcg(reinterpret_cast<const float2*>(tp + 2 * tig + 8));
          tv[0] = v01.x; tv[1] = v01.y; tv[2] = v89.x; tv[3] = v89.y;
          uint32_t hi[2], lo[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int rank0 = 16 * c + 2 * tig + 8 * h;
            const float ta = (rank0 < m.r) ? tv[2 * h] : 0.f;
            const float tb = (rank0 + 1 < m.r) ? tv[2 * h + 1] : 0.f;
            const uint32_t ha = f32_to_bf16_rn(ta), hb = f32_to_bf16_rn(tb);
            hi[h] = ha | (hb << 16);
            lo[h] = f32_to_bf16_rn(ta - bf16_bits_to_f32(ha)) | (f32_to_bf16_rn(tb - bf16_bits_to_f32(hb)) << 16);
          }
          mma16816(comp[nb], af, hi[0], hi[1]);
          mma16816(comp[nb], af, lo[0], lo[1]);
        }
      }
    }
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int b = 2 * tig + (e & 1) + 8 * nb;
        if (b >= a.B) continue;
        const int n = m.row_off + rbl * kRows + gid + 8 * (e >> 1);
        float v = fin[nb][e] + comp[nb][e];
        if (a.resid) v += bf16_bits_to_f32(a.resid[(size_t)b * a.ld_resid + n]);
        if (a.y_bf16)
          reinterpret_cast<uint16_t*>(a.y)[(size_t)b * a.ldy + n] = (uint16_t)f32_to_bf16_rn(v);
        else
          reinterpret_cast<float*>(a.y)[(size_t)b * a.ldy + n] = v;
      }
    __syncwarp();
    if (lane == 0) {
      const unsigned old = atomicAdd(&a.cnt[a.n_chunks + 1], 1u);
      if (old == (unsigned)a.n_rb - 1) {       // last row block of the launch: reset counters
        a.cnt[a.n_chunks] = 0u;
        a.cnt[a.n_chunks + 1] = 0u;
      }
    }
  }
}

static size_t decode_smem_bytes() {
  return (size_t)kDecodeWarps * kRing * kSlotBytes + 2 * kDecodeWarps * 32 * 8 * sizeof(float) +
         kDecodeWarps * kRing * sizeof(uint64_t);
}

template <int BITS, int NB8>
static cudaError_t launch_t(const DArgs& a, int grid, cudaStream_t st) {
  const size_t smem = decode_smem_bytes();
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<BITS, NB8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  decode_kernel<BITS, NB8><<<grid, kDecodeWarps * 32, smem, st>>>(a);
  return cudaGetLastError();
}

template <int BITS, int NB8>
static int max_ctas_t() {
  const size_t smem = decode_smem_bytes();
  cudaFuncSetAttribute(decode_kernel<BITS, NB8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0, dev = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<BITS, NB8>, kDecodeWarps * 32, smem);
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}

cudaError_t launch_decode(const DArgs& a, int bits, int grid, cudaStream_t st) {
  const bool two = a.B > 8;
  switch (bits) {
    case 2: return two ? launch_t<2, 2>(a, grid, st) : launch_t<2, 1>(a, grid, st);
    case 3: return two ? launch_t<3, 2>(a, grid, st) : launch_t<3, 1>(a, grid, st);
    case 4: return two ? launch_t<4, 2>(a, grid, st) : launch_t<4, 1>(a, grid, st);
    default: return cudaErrorInvalidValue;
  }
}

int decode_max_ctas(int bits, int B) {
  const bool two = B > 8;
  switch (bits) {
    case 2: return two ? max_ctas_t<2, 2>() : max_ctas_t<2, 1>();
    case 3: return two ? max_ctas_t<3, 2>() : max_ctas_t<3, 1>();
    case 4: return two ? max_ctas_t<4, 2>() : max_ctas_t<4, 1>();
    default: return 0;
  }
}

}  // namespace hc
