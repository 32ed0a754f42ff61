// Prefill compensated GEMM on 5th-generation tensor cores (tcgen05 + TMEM + TMA + mbarriers).
//
//     Y[m][n] = Σ_k X[m][k] · s[n][k/128]·(q[n][k] − z[n][k/128])  +  Σ_j T[m][j] · U[n][j],
//     T = X · V[:r]ᵀ
//
// i.e. Y = [X | T] · [deq(W) | U]ᵀ: the rank-r update is appended to the K loop and lands in the
// same TMEM accumulator.  One CTA computes a 128 (tokens) x 256 (weight rows) tile:
//   warp 0      TMA producer: X tiles (and T / U tiles for the rank slice, V tiles for T = X·Vᵀ)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (kind::f16, M=128, N<=256, K=16)
//   warps 2-9   dequant producers: 4-bit codes -> fp16 s·(q−z) written straight into the UMMA
//               K-major 128-byte-swizzled smem layout (exact (q−z), one fp16 rounding of s·(q−z))
//   warps 10-13 epilogue: tcgen05.ld TMEM -> registers -> fp32 / bf16 / fp16 global stores
// 3-stage smem ring (~57 KB per stage) with full/empty mbarriers; tcgen05.commit releases stages.
// Persistent CTAs (one per SM) loop over tiles; the TMEM accumulator is double-buffered (2 x 256
// columns) with tmem_full / tmem_empty barriers, so a tile's epilogue overlaps the next main loop.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include "layout.h"
#include "prefill.h"

namespace hc {

namespace {

constexpr int kABytes = kPBM * kPBK * 2;   // 16 KB
constexpr int kBBytes = kPBN * kPBK * 2;   // 32 KB
constexpr int kCBytes = kPBN * kPBK / 2;   // 8 KB of 4-bit codes per stage
constexpr int kSBytes = kPBN * 2;          // bf16 scales of the stage's group
constexpr int kZBytes = kPBN;              // zeros
#ifndef HC_PF_DQW
#define HC_PF_DQW 8
#endif
constexpr int kDqWarps = HC_PF_DQW;        // dequant producer warps (4 or 8): rows per thread = 256 / (32·kDqWarps)
constexpr int kThreads = (2 + kDqWarps + 4) * 32;

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(s_u32(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(b)) : "memory");
}
__device__ __forceinline__ void bulk_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(s_u32(dst)),
               "l"(src), "r"(bytes), "r"(s_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(s_u32(dst)),
      "l"(map), "r"(s_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// UMMA shared-memory descriptor: K-major, 128-byte swizzle, 8-row atoms 1024 B apart (SBO),
// sm100 descriptor version 1.
__device__ __forceinline__ uint64_t umma_desc(const void* smem) {
  const uint64_t addr = s_u32(smem);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;                 // start address
  d |= (uint64_t)(16 >> 4) << 16;               // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;             // SBO
  d |= (uint64_t)1 << 46;                       // version (sm100)
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: A = B = F16 (K-major), D = F32, M = 128, N = n.
__device__ __forceinline__ uint32_t umma_idesc(int n) {
  uint32_t d = 0;
  d |= 1u << 4;                                 // D format F32
  d |= 0u << 7;                                 // A F16
  d |= 0u << 10;                                // B F16
  d |= (uint32_t)(n >> 3) << 17;                // N >> 3
  d |= (uint32_t)(kPBM >> 4) << 24;             // M >> 4
  return d;
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(bar))
               : "memory");
}

// byte offset of (row, 16-byte chunk) inside a K-major SW128 tile (rows of 128 B, 8-row atoms)
__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
  return ((row >> 3) << 10) + ((row & 7) << 7) + (((chunk ^ row) & 7) << 4);
}

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

}  // namespace

// Work item w (persistent loop): tile = w % n_tiles (M-fastest, so the CTAs running concurrently
// share weight tiles through L2), split-K slice ks = w / n_tiles.
struct TileWork {
  int m0, n0, ks, kb_lo, nkb1, nkb;
};
__device__ __forceinline__ TileWork tile_work(const PArgs& p, int w) {
  TileWork t;
  const int n_tiles = p.tiles_m * p.tiles_n;
  const int tile = w % n_tiles;
  t.ks = w / n_tiles;
  t.m0 = (tile % p.tiles_m) * kPBM;
  t.n0 = (tile / p.tiles_m) * kPBN;
  const int nkb_all = p.K / kPBK;
  t.kb_lo = t.ks * nkb_all / p.ksplit;
  t.nkb1 = (t.ks + 1) * nkb_all / p.ksplit - t.kb_lo;
  t.nkb = t.nkb1 + (p.K2 + kPBK - 1) / kPBK;
  return t;
}

// Persistent: each CTA loops over work items; the producer / MMA / dequant roles run one continuous
// stage sequence across tiles, and the accumulator is double-buffered in TMEM (2 x 256 columns) so
// the epilogue of tile j overlaps the main loop of tile j + 1.
__global__ void __launch_bounds__(kThreads, 1)
    prefill_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ PArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = base;
  uint8_t* sB = sA + kPStages * kABytes;
  uint8_t* sC = sB + kPStages * kBBytes;
  uint8_t* sS = sC + kPStages * kCBytes;
  uint8_t* sZ = sS + kPStages * kSBytes;
  uint64_t* full_a = reinterpret_cast<uint64_t*>(sZ + kPStages * kZBytes);
  uint64_t* full_b = full_a + kPStages;
  uint64_t* empty = full_b + kPStages;
  uint64_t* tmem_full = empty + kPStages;      // [2]
  uint64_t* tmem_empty = tmem_full + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_work = p.tiles_m * p.tiles_n * p.ksplit;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      bar_init(&full_a[s], 1);
      bar_init(&full_b[s], kDqWarps * 32);
      bar_init(&empty[s], 1);
    }
    bar_init(&tmem_full[0], 1); bar_init(&tmem_full[1], 1);
    bar_init(&tmem_empty[0], 4); bar_init(&tmem_empty[1], 4);   // one arrive per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s_u32(tmem_slot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      int ig = 0;                                   // global stage counter of this CTA
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        const TileWork tw = tile_work(p, w);
        for (int i = 0; i < tw.nkb; ++i, ++ig) {
          const int s = ig % kPStages;
          if (ig >= kPStages) bar_wait(&empty[s], ((ig / kPStages) + 1) & 1);
          const bool main = i < tw.nkb1;
          const int kb = tw.kb_lo + i;
          if (main && p.b_mode == 0) {
            // X tile + this k-block's codes (256 rows x 32 B) + the group's scales and zeros
            bar_expect_tx(&full_a[s], (uint32_t)(kABytes + kCBytes + kSBytes + kZBytes));
            tma_2d(sA + s * kABytes, &tmA, kb * kPBK, tw.m0, &full_a[s]);
            tma_2d(sC + s * kCBytes, &tmC, kb * (kPBK / 8), tw.n0, &full_a[s]);
            const int g = kb >> 1;
            bulk_1d(sS + s * kSBytes, p.scales_t + (size_t)g * p.N + tw.n0, kSBytes, &full_a[s]);
            bulk_1d(sZ + s * kZBytes, p.zeros_t + (size_t)g * p.N + tw.n0, kZBytes, &full_a[s]);
          } else if (main) {
            bar_expect_tx(&full_a[s], (uint32_t)(kABytes + kBBytes));
            tma_2d(sA + s * kABytes, &tmA, kb * kPBK, tw.m0, &full_a[s]);
            tma_2d(sB + s * kBBytes, &tmB, kb * kPBK, tw.n0, &full_a[s]);
          } else {
            bar_expect_tx(&full_a[s], (uint32_t)(kABytes + kBBytes));
            tma_2d(sA + s * kABytes, &tmA2, (i - tw.nkb1) * kPBK, tw.m0, &full_a[s]);
            tma_2d(sB + s * kBBytes, &tmB2, (i - tw.nkb1) * kPBK, tw.n0, &full_a[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (one thread) =======================
    if (lane == 0) {
      const uint32_t idesc = umma_idesc(p.n_dim);
      int ig = 0, j = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++j) {
        const TileWork tw = tile_work(p, w);
        const int buf = j & 1;
        if (j >= 2) bar_wait(&tmem_empty[buf], ((j >> 1) + 1) & 1);   // epilogue of tile j - 2 drained it
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem_base + (uint32_t)(buf * kPBN);
        for (int i = 0; i < tw.nkb; ++i, ++ig) {
          const int s = ig % kPStages;
          const uint32_t ph = (ig / kPStages) & 1;
          bar_wait(&full_a[s], ph);
          bar_wait(&full_b[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int nk = i < tw.nkb1 ? kPBK / 16 : min(kPBK, p.K2 - (i - tw.nkb1) * kPBK) / 16;
          const uint64_t ad = umma_desc(sA + s * kABytes), bd = umma_desc(sB + s * kBBytes);
          for (int k = 0; k < nk; ++k)   // advance 16 fp16 = 32 bytes along K inside the swizzled rows
            umma_f16(acc, ad + (uint64_t)(2 * k), bd + (uint64_t)(2 * k), idesc, (i | k) != 0);
          umma_commit(&empty[s]);
        }
        umma_commit(&tmem_full[buf]);
      }
    }
  } else if (warp < 2 + kDqWarps) {
    // ======================= dequant producers (smem -> smem) =======================
    const int t = threadIdx.x - 64;            // rows t, t + 32·kDqWarps, ... of the B tile
    int ig = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
      const TileWork tw = tile_work(p, w);
      for (int i = 0; i < tw.nkb; ++i, ++ig) {
        const int s = ig % kPStages;
        bar_wait(&full_a[s], (ig / kPStages) & 1);   // codes of this stage landed (and stage s is free)
        if (i < tw.nkb1 && p.b_mode == 0) {
          uint8_t* tile = sB + s * kBBytes;
          const uint8_t* codes = sC + s * kCBytes;
#pragma unroll
          for (int h = 0; h < 256 / (32 * kDqWarps); ++h) {
            const int row = t + 32 * kDqWarps * h;
            const uint4 c0 = *reinterpret_cast<const uint4*>(codes + row * 32);
            const uint4 c1 = *reinterpret_cast<const uint4*>(codes + row * 32 + 16);
            const uint32_t words[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
            const float sf = __uint_as_float((uint32_t)reinterpret_cast<const uint16_t*>(sS + s * kSBytes)[row] << 16);
            const uint32_t sc = (uint32_t)__half_as_ushort(__float2half_rn(sf)) * 0x00010001u;      // half2(s, s)
            const uint32_t zz = (0x6400u + (uint32_t)(sZ + s * kZBytes)[row]) * 0x00010001u;       // half2(1024+z)
#pragma unroll
            for (int c = 0; c < 8; ++c) {        // word c = k 8c..8c+7 = 16-byte chunk c of the row
              uint32_t v[4];
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                uint32_t hv = lop3_and_or(words[c] >> (4 * jj), 0x000F000Fu, 0x64006400u);   // half2(1024 + q)
                __half2 d = __hsub2(*reinterpret_cast<__half2*>(&hv), *reinterpret_cast<const __half2*>(&zz));
                d = __hmul2(d, *reinterpret_cast<const __half2*>(&sc));                       // fp16(s·(q − z))
                v[jj] = *reinterpret_cast<uint32_t*>(&d);
              }
              *reinterpret_cast<uint4*>(tile + sw128(row, c)) = make_uint4(v[0], v[1], v[2], v[3]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
        }
        bar_arrive(&full_b[s]);
      }
    }
  } else {
    // ======================= epilogue =======================
    const int q = warp & 3;                    // TMEM lane quadrant this warp may access
    int j = 0;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x, ++j) {
      const TileWork tw = tile_work(p, w);
      const int buf = j & 1;
      const int m = tw.m0 + 32 * q + lane;
      bar_wait(&tmem_full[buf], (j >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      void* outp = p.ksplit > 1 ? (void*)(reinterpret_cast<float*>(p.out) + (size_t)tw.ks * p.M * p.ldo) : p.out;
      for (int c0 = 0; c0 < p.n_dim; c0 += 32) {
        uint32_t v[32];
        const uint32_t addr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * kPBN + c0);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
              "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(addr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int n = tw.n0 + c0;
        if (m < p.M && n < p.N) {
          if (p.rsig) {                                // the row's X prescale (exact power of two, R20)
            const float rs = __ldg(p.rsig + m);
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * rs);
          }
          if (p.out_type == 0) {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(outp) + (size_t)m * p.ldo + n);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              dst[i] = make_float4(__uint_as_float(v[4 * i]), __uint_as_float(v[4 * i + 1]),
                                   __uint_as_float(v[4 * i + 2]), __uint_as_float(v[4 * i + 3]));
          } else {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float a = __uint_as_float(v[2 * i]), b = __uint_as_float(v[2 * i + 1]);
              if (p.out_type == 1) {
                __nv_bfloat162 h2 = __floats2bfloat162_rn(a, b);
                pk[i] = *reinterpret_cast<uint32_t*>(&h2);
              } else {
                __half2 h2 = __floats2half2_rn(a, b);
                pk[i] = *reinterpret_cast<uint32_t*>(&h2);
              }
            }
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(outp) + (size_t)m * p.ldo + n);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) bar_arrive(&tmem_empty[buf]);   // this warp's quadrant of buffer buf is drained
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
  }
}

static size_t prefill_smem() {
  return (size_t)kPStages * (kABytes + kBBytes + kCBytes + kSBytes + kZBytes) + (3 * kPStages + 5) * 8 + 1024;
}

cudaError_t launch_prefill(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA2,
                           const CUtensorMap& tmB2, const CUtensorMap& tmC, const PArgs& p, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prefill_smem());
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int n_work = p.tiles_m * p.tiles_n * p.ksplit;
  const int grid = n_work < sms ? n_work : sms;      // persistent: one CTA per SM (smem-limited)
  prefill_kernel<<<grid, kThreads, prefill_smem(), st>>>(tmA, tmB, tmA2, tmB2, tmC, p);
  return cudaGetLastError();
}

__global__ void splitk_reduce_kernel(const float* __restrict__ part, int ksplit, size_t n, uint16_t* __restrict__ out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc = 0.f;
  for (int k = 0; k < ksplit; ++k) acc += part[(size_t)k * n + i];   // fixed order: deterministic
  out[i] = __half_as_ushort(__float2half_rn(acc));
}

cudaError_t launch_splitk_reduce_f16(const float* partial, int ksplit, int M, int ld, uint16_t* out, cudaStream_t st) {
  const size_t n = (size_t)M * ld;
  splitk_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(partial, ksplit, n, out);
  return cudaGetLastError();
}

__global__ void transpose_groups_kernel(const uint16_t* __restrict__ s_in, const uint8_t* __restrict__ z_in, int rows,
                                        int G, uint16_t* __restrict__ s_out, uint8_t* __restrict__ z_out) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (size_t)rows * G) return;
  const int r = (int)(i / G), g = (int)(i % G);
  s_out[(size_t)g * rows + r] = s_in[i];
  z_out[(size_t)g * rows + r] = z_in[i];
}

cudaError_t launch_transpose_groups(const uint16_t* s_in, const uint8_t* z_in, int rows, int G, uint16_t* s_out,
                                    uint8_t* z_out, cudaStream_t st) {
  const size_t n = (size_t)rows * G;
  transpose_groups_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s_in, z_in, rows, G, s_out, z_out);
  return cudaGetLastError();
}

bool encode_tmap_codes(CUtensorMap* map, const void* base, uint64_t words_per_row, uint64_t rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return false;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  const cuuint64_t dims[2] = {words_per_row, rows};
  const cuuint64_t strides[1] = {words_per_row * 4};
  const cuuint32_t box[2] = {8, 256};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__global__ void bf16_to_f16_kernel(const uint16_t* __restrict__ in, uint16_t* __restrict__ out, size_t n) {
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (i + 8 <= n) {
    const uint4 v = *reinterpret_cast<const uint4*>(in + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float a = __uint_as_float(w[j] << 16), b = __uint_as_float(w[j] & 0xFFFF0000u);
      __half2 h = __floats2half2_rn(a, b);
      o[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(out + i) = make_uint4(o[0], o[1], o[2], o[3]);
  } else {
    for (size_t j = i; j < n; ++j) out[j] = __half_as_ushort(__float2half_rn(__uint_as_float((uint32_t)in[j] << 16)));
  }
}

// X (bf16 [M][K]) -> X' = X·2^-σ_m (fp16), one CTA per token row m, and rsig[m] = 2^σ_m (R20,
// prefill form: one power of two per row, because the tcgen05 accumulator spans all of K).  σ_m = 0 when
// the row's largest |x| has exponent E in [-2, 13] (exactly the plain conversion), else E - 8 (clamped to
// [-100, 115]): X' then holds every bf16 x within 2^25 of the row maximum exactly, for any bf16 range.
// The T = X'·Vᵀ slice is in the same scaled units, so the epilogue's factor 2^σ_m restores the whole row.
__global__ void __launch_bounds__(256) x_rows_f16_kernel(const uint16_t* __restrict__ in, int K, uint16_t* __restrict__ out,
                                                         float* __restrict__ rsig) {
  __shared__ uint32_t wmax[8];
  const int m = blockIdx.x;
  const uint16_t* row = in + (size_t)m * K;
  uint32_t mx = 0;
  for (int i = threadIdx.x * 8; i < K; i += 256 * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(row + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) mx = max(mx, max(w[j] & 0x7FFFu, (w[j] >> 16) & 0x7FFFu));
  }
  mx = __reduce_max_sync(0xFFFFFFFFu, mx);
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) mx = max(mx, wmax[w]);
  int sig = 0;
  if (mx != 0 && mx < 0x7F80u) {
    const int E = max((int)(mx >> 7), 1) - 127;
    if (E < -2 || E > 13) sig = min(max(E - 8, -100), 115);
  }
  const float ps = __uint_as_float((uint32_t)(127 - sig) << 23);
  for (int i = threadIdx.x * 8; i < K; i += 256 * 8) {
    const uint4 v = *reinterpret_cast<const uint4*>(row + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      __half2 h = __floats2half2_rn(__uint_as_float(w[j] << 16) * ps, __uint_as_float(w[j] & 0xFFFF0000u) * ps);
      o[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(out + (size_t)m * K + i) = make_uint4(o[0], o[1], o[2], o[3]);
  }
  if (threadIdx.x == 0) rsig[m] = __uint_as_float((uint32_t)(127 + sig) << 23);
}

cudaError_t launch_x_rows_f16(const uint16_t* in, int M, int K, uint16_t* out, float* rsig, cudaStream_t st) {
  if (K % 8) return cudaErrorInvalidValue;
  x_rows_f16_kernel<<<M, 256, 0, st>>>(in, K, out, rsig);
  return cudaGetLastError();
}

cudaError_t launch_bf16_to_f16(const uint16_t* in, uint16_t* out, size_t n, cudaStream_t st) {
  const size_t threads = (n + 7) / 8;
  bf16_to_f16_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

// word w of a row (elements 8w..8w+7, canonical nibble j = element 8w+j) -> prefill order:
// nibble 0 = k0, 4 = k1, 1 = k2, 5 = k3, 2 = k4, 6 = k5, 3 = k6, 7 = k7 (so that (w >> 4i) & 0x000F000F
// is the fp16 pair (k_{2i}, k_{2i+1}))
__global__ void prefill_codes_kernel(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, size_t n) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t w = in[i];
  uint32_t o = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int pos = (j >> 1) + 4 * (j & 1);
    o |= ((w >> (4 * j)) & 0xFu) << (4 * pos);
  }
  out[i] = o;
}

cudaError_t launch_prefill_codes(const uint32_t* canon, uint32_t* out, size_t n_words, cudaStream_t st) {
  prefill_codes_kernel<<<(unsigned)((n_words + 255) / 256), 256, 0, st>>>(canon, out, n_words);
  return cudaGetLastError();
}

bool encode_tmap_f16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                     uint32_t box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !f)
      return false;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace hc
