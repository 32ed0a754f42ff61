// Grouped MoE expert path (C3).
//
//   y[t] = Σ_j g[t,j] · DOWN_e(m_e),  m_e = bf16(silu(GATE_e(x_t)) ⊙ UP_e(x_t)),  e = topk_idx[t,j],
//   every product compensated at its own rank (north_star; oracle.linear.moe_forward).
//
// Pipeline (one launch each, all activated experts of the layer together — the paper's cross-expert
// window fusion on the GPU instead of one CPU task per expert):
//   route     group the T·k (token, expert) pairs by expert (ascending), tokens ascending inside an
//             expert; entries = chunks of <= 16 rows of one expert (the mma N dimension)
//   prep      gather x rows per (token, expert) row: bf16 copy (for V·x) and x' = x·2^-fp (fp16)
//   rank_proj t[row] = V_e·x_row with the natural-k V fragments (one block per entry, member, 16 ranks;
//             8 warps split K, fixed-order reduction: deterministic)
//   gemv      one warp per (entry, row block) over all K groups: records decoded exactly as the
//             decode kernel does (w_tile_regs; the next record's words load while one is decoded),
//             U·t (bf16 hi + lo) and the SiLU glue in the same warp — no reduction, no barrier
//   combine   y[t] = Σ_j g[t,j]·dout[row(t,j)] in slot order j
#include <cuda_bf16.h>

#include "decode_dev.cuh"
#include "moe.h"

namespace hc {

namespace {

constexpr int kRouteThreads = 1024;

// Single CTA: T <= 1024 tokens, E <= 256 experts, k <= 16.  Per-expert token bitmaps (order-free
// atomicOr), per-expert counts and entry counts by one thread per expert, exclusive scans over the
// experts (one warp, fixed order), then every (token, slot) finds its row by popcount.
// Align (ties up) and the cap rule (R15) of the oracle on the continuous rank
// rt = (k·g)·r̃, which is EXACT in float64 (k <= 16: 5 bits, g and r̃ fp32: 24 bits each -> <= 53 bits), so
// the integer decision is exact and equal to the oracle's.  Bounded for any finite or infinite rt: with
// L = the largest level <= cap, an rt >= L aligns to a level >= L, which the cap maps to L.
__device__ __forceinline__ int dyn_rank(double rt, int cap, int k0) {
  int L = 0;
  for (int v = 1 << k0; v <= cap && v <= (1 << 30); v *= 2) L = v;
  if (!(rt < (double)L)) return L;                // rt >= L (also inf; NaN is rejected at the ABI)
  int lo = 0, hi = 1 << k0;
  while (rt >= (double)hi) { lo = hi; hi *= 2; }  // hi <= L <= 2^30: terminates
  return (rt - (double)lo) < ((double)hi - rt) ? lo : hi;
}

__global__ void moe_route_kernel(const int32_t* __restrict__ idx, const float* __restrict__ gate, int T, int k, int E,
                                 MoERoute rt, MoEDyn dyn) {
  asm volatile("griddepcontrol.wait;" ::: "memory");                 // PDL: the previous launch's outputs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ unsigned bm[];                 // [E][W] token bitmaps, W = ceil(T/32)
  __shared__ int cnt[256], ecnt[256], off[257], eoff[257];
  const int W = (T + 31) / 32;
  for (int i = threadIdx.x; i < E * W; i += blockDim.x) bm[i] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < T * k; i += blockDim.x) {
    const int e = idx[i], t = i / k;
    if (e >= 0 && e < E) atomicOr(&bm[e * W + (t >> 5)], 1u << (t & 31));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    int c = 0;
    for (int w = 0; w < W; ++w) c += __popc(bm[e * W + w]);
    cnt[e] = c;
    ecnt[e] = (c + 15) / 16;
  }
  __syncthreads();
  if (threadIdx.x < 32) {                          // exclusive scans of cnt and ecnt (E <= 256)
    const int lane = threadIdx.x;
    int base_r = 0, base_e = 0;
    for (int e0 = 0; e0 < E; e0 += 32) {
      const int e = e0 + lane;
      int vr = e < E ? cnt[e] : 0, ve = e < E ? ecnt[e] : 0;
      int sr = vr, se = ve;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tr = __shfl_up_sync(0xffffffffu, sr, o), te = __shfl_up_sync(0xffffffffu, se, o);
        if (lane >= o) { sr += tr; se += te; }
      }
      if (e < E) { off[e] = base_r + sr - vr; eoff[e] = base_e + se - ve; }
      base_r += __shfl_sync(0xffffffffu, sr, 31);
      base_e += __shfl_sync(0xffffffffu, se, 31);
    }
    if (lane == 0) { off[E] = base_r; eoff[E] = base_e; *rt.n_rows = base_r; *rt.n_ent = base_e; }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    for (int j = 0; j < ecnt[e]; ++j) {
      const int ne = eoff[e] + j;
      rt.ent_e[ne] = e;
      rt.ent_row0[ne] = off[e] + 16 * j;
      rt.ent_ncol[ne] = min(16, cnt[e] - 16 * j);
    }
  for (int i = threadIdx.x; i < T * k; i += blockDim.x) {
    const int e = idx[i], t = i / k;
    if (e < 0 || e >= E) { rt.tok_row[i] = -1; continue; }
    int before = 0;                                 // tokens < t routed to e
    for (int w = 0; w < (t >> 5); ++w) before += __popc(bm[e * W + w]);
    before += __popc(bm[e * W + (t >> 5)] & ((1u << (t & 31)) - 1u));
    const int row = off[e] + before;
    rt.row_tok[row] = t;
    rt.tok_row[i] = row;
    if (dyn.row_rank) {
      const double kg = (double)k * (double)gate[i];             // G = k·g (exact in float64)
#pragma unroll
      for (int sl = 0; sl < 3; ++sl)
        dyn.row_rank[row * 3 + sl] = (uint16_t)dyn_rank(kg * (double)dyn.rtilde[e * 3 + sl], dyn.caps[e * 3 + sl], dyn.k0);
    }
  }
}

template <int BITS>
__global__ void moe_prep_kernel(const uint16_t* __restrict__ x, int ldx, int K, int gather, MoERoute rt, int R_max,
                                uint16_t* __restrict__ xg, uint16_t* __restrict__ x16, float* __restrict__ xsig) {
  asm volatile("griddepcontrol.wait;" ::: "memory");                 // PDL: the previous launch's outputs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // one thread per (row, 16-element part); the 8 parts of a (row, group) are 8 consecutive lanes (K/16 is
  // a multiple of 8) and agree on the group's B-operand prescale σ (R20): 2^σ -> xsig[row][g]
  const int parts = K / 16;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)R_max * parts) return;
  const int r = (int)(i / parts), p = (int)(i % parts);
  if (r >= *rt.n_rows) return;                      // uniform per 8-lane group (a whole row)
  const int src = gather ? rt.row_tok[r] : r;
  const uint4* s = reinterpret_cast<const uint4*>(x + (size_t)src * ldx + p * 16);
  const uint4 in[2] = {s[0], s[1]};
  if (gather) {
    uint4* d = reinterpret_cast<uint4*>(xg + (size_t)r * K + p * 16);
    d[0] = in[0]; d[1] = in[1];
  }
  const unsigned m8 = 0xFFu << (threadIdx.x & 24);
  uint32_t m = max(absmax8(in[0]), absmax8(in[1]));
  m = max(m, __shfl_xor_sync(m8, m, 1));
  m = max(m, __shfl_xor_sync(m8, m, 2));
  m = max(m, __shfl_xor_sync(m8, m, 4));
  const int sig = prescale_sigma(m);
  uint4 out[2];
  xprime16<BITS>(in, p & 7, out, sig);              // 16-element part p & 7 of group p / 8
  uint4* d = reinterpret_cast<uint4*>(x16 + (size_t)r * K + p * 16);
  d[0] = out[0]; d[1] = out[1];
  if ((p & 7) == 0) xsig[(size_t)r * (K / kGroup) + (p >> 3)] = pow2i(sig);
}

// one block of kRPW warps per (entry, member, 16-rank chunk); warp w takes k-blocks [w·KB/kRPW, (w+1)·KB/kRPW)
// (up to 8 in flight, independent loads: the whole V slice of a job is requested in about one round trip),
// partials summed in a fixed order through shared memory.  (8 warps with 4 loads in flight: 12.6 µs for the C3
// UPGATE projection at T = 1, latency-bound on 18 CTAs.)
// warps per rank-projection job: 16 when the jobs are few (T = 1: 18 CTAs, latency-bound; measured C3 T = 1
// 545 -> 583 tokens/s), 8 when they fill the GPU (T = 256: 16 warps measured -3%)
template <int kRPW>
__global__ void __launch_bounds__(kRPW * 32) moe_rank_proj_kernel(MoEWin w, MoERoute rt, int max_ent, int max_chunks,
                                                            const uint16_t* __restrict__ xg, float* __restrict__ t) {
  asm volatile("griddepcontrol.wait;" ::: "memory");                 // PDL: the previous launch's outputs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ float part[kRPW][32][8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const int job = blockIdx.x, per_ent = 2 * max_chunks;
  const int ent = job / per_ent, rem = job % per_ent, mb = rem / max_chunks, c = rem % max_chunks;
  if (ent >= *rt.n_ent || (mb == 1 && !w.glue)) return;      // uniform per block
  const MoEExpert& ex = w.ex[rt.ent_e[ent]];
  if (16 * c >= ex.r[mb]) return;
  const int row0 = rt.ent_row0[ent], ncol = rt.ent_ncol[ent];
  const int cs = ex.rs[mb] / 16;
  const uint4* vn = ex.Vn[mb];
  const int KB = w.K / 16, kb_lo = warp * KB / kRPW, kb_hi = (warp + 1) * KB / kRPW;
  const uint16_t* xr0[2];
  bool cv[2];
#pragma unroll
  for (int nb = 0; nb < 2; ++nb) {
    const int col = gid + 8 * nb;
    cv[nb] = col < ncol;
    xr0[nb] = xg + (size_t)(row0 + (cv[nb] ? col : 0)) * w.K + 2 * tig;
  }
  constexpr int U = 4, NCH = 4;                          // loads in flight per warp, independent mma chains
  float acc[NCH][2][4] = {};
  for (int kb0 = kb_lo; kb0 < kb_hi; kb0 += U) {
    uint4 a4[U];
    uint32_t b[U][2][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kb = min(kb0 + u, kb_hi - 1);
      a4[u] = __ldg(vn + ((size_t)kb * cs + c) * 32 + lane);
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        b[u][nb][0] = cv[nb] ? __ldg(reinterpret_cast<const uint32_t*>(xr0[nb] + 16 * kb)) : 0u;
        b[u][nb][1] = cv[nb] ? __ldg(reinterpret_cast<const uint32_t*>(xr0[nb] + 16 * kb + 8)) : 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kb0 + u >= kb_hi) break;
      const uint32_t af[4] = {a4[u].x, a4[u].y, a4[u].z, a4[u].w};
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) mma16816(acc[u % NCH][nb], af, b[u][nb][0], b[u][nb][1]);
    }
  }
#pragma unroll
  for (int nb = 0; nb < 2; ++nb)
#pragma unroll
    for (int e = 0; e < 4; ++e)
      {
        float v = acc[0][nb][e];
#pragma unroll
        for (int q = 1; q < NCH; ++q) v += acc[q][nb][e];
        part[warp][lane][4 * nb + e] = v;
      }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        float v = 0.f;
        for (int ww = 0; ww < kRPW; ++ww) v += part[ww][lane][4 * nb + e];   // fixed order
        const int col = 2 * tig + (e & 1) + 8 * nb, rank = 16 * c + gid + 8 * (e >> 1);
        if (col < ncol && rank < ex.r[mb]) t[(size_t)(row0 + col) * w.t_ld + mb * (w.t_ld / 2) + rank] = v;
      }
  }
}

// One warp per (entry, row block) over all K: no cross-warp reduction, no CTA barrier; the next
// record's words are loaded while the current one is decoded (many warps per SM hide the rest).
// KS: the item's K groups are split over the CTA's 4 warps (few items: routing of a handful of
// tokens); else every warp owns whole items (many items).
constexpr int kKSW = 4;   // K-split items: warps per CTA (8 measured slower: C3 T = 1 579 -> 463 tokens/s)
template <int BITS, int NB8, bool KS>
__global__ void __launch_bounds__(KS ? kKSW * 32 : 128) moe_gemv_warp_kernel(MoEWin w, MoERoute rt, const uint16_t* __restrict__ x16,
                                                           const float* __restrict__ xsig, const float* __restrict__ t,
                                                           void* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");                 // PDL: the previous launch's outputs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // one (entry, row block) item per CTA; its K groups split over the kKSW warps (each warp keeps one
  // record in flight ahead of the one it decodes), partials summed in a fixed order by warp 0
  __shared__ float red[KS ? kKSW : 1][32][4 * NB8];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  const long long n_items = (long long)(*rt.n_ent) * w.n_rb;
  const long long it0 = KS ? (long long)blockIdx.x : (long long)blockIdx.x * 4 + warp;
  const long long its = KS ? (long long)gridDim.x : (long long)gridDim.x * 4;
  for (long long it = it0; it < n_items; it += its) {
    const int ent = (int)(it / w.n_rb), rb = (int)(it % w.n_rb);
    const MoEExpert& ex = w.ex[rt.ent_e[ent]];
    const int row0 = rt.ent_row0[ent], ncol = rt.ent_ncol[ent];
    const uint8_t* rec0 = ex.rec + (size_t)rb * w.G * rec_bytes(BITS);
    float tot[NB8][4];
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) tot[nb][e] = 0.f;
    const uint16_t* xrow[NB8];
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb) {
      const int col = gid + 8 * nb;
      xrow[nb] = x16 + (size_t)(row0 + (col < ncol ? col : 0)) * w.K + 8 * tig;
    }
    const int g_lo = KS ? warp * w.G / kKSW : 0, g_hi = KS ? (warp + 1) * w.G / kKSW : w.G;
    uint32_t wn[2 * BITS], swn;
    uint2 zzn;
    if (g_lo < g_hi) load_record<BITS>(rec0 + (size_t)g_lo * rec_bytes(BITS), lane, wn, swn, zzn);
    for (int g = g_lo; g < g_hi; ++g) {
      uint32_t wc[2 * BITS];
#pragma unroll
      for (int i = 0; i < 2 * BITS; ++i) wc[i] = wn[i];
      const uint32_t swc = swn;
      const uint2 zzc = zzn;
      if (g + 1 < g_hi) load_record<BITS>(rec0 + (size_t)(g + 1) * rec_bytes(BITS), lane, wn, swn, zzn);
      uint32_t xr[NB8][16];
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb) {
        const uint4* p = reinterpret_cast<const uint4*>(xrow[nb] + g * kGroup);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint4 v = __ldg(p + 4 * q);
          xr[nb][4 * q + 0] = v.x; xr[nb][4 * q + 1] = v.y; xr[nb][4 * q + 2] = v.z; xr[nb][4 * q + 3] = v.w;
        }
      }
      const uint4* unused[NB8] = {};
      float fs[NB8][2];                               // 2^σ of the lane's output columns (rows of this entry)
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 2 * tig + h + 8 * nb;
          fs[nb][h] = __ldg(xsig + (size_t)(row0 + (col < ncol ? col : 0)) * w.G + g);
        }
      w_tile_regs<BITS, NB8, false, true>(wc, swc, zzc, lane, unused, xr, tot, fs);
    }
    if constexpr (KS) {
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
        *reinterpret_cast<float4*>(&red[warp][lane][4 * nb]) = make_float4(tot[nb][0], tot[nb][1], tot[nb][2], tot[nb][3]);
      __syncthreads();
      if (warp == 0) {
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float v = red[0][lane][4 * nb + e];
#pragma unroll
            for (int q = 1; q < kKSW; ++q) v += red[q][lane][4 * nb + e];   // fixed order: deterministic
            tot[nb][e] = v;
          }
      }
    }
    // K-split items: warp 0 finishes the item; every warp meets the same barrier below (red is reused)
    if (!KS || warp == 0) {
    // U·t (plain: member 0 on all 16 rows; SiLU window: up chunks on rows 0-7 with t of member 0,
    // gate chunks on rows 8-15 with t of member 1), then the glue and the output
    float comp[2][NB8][4];
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) comp[h][nb][e] = 0.f;
    const int r_eff = w.glue ? max(ex.r[0], ex.r[1]) : ex.r[0];
    const int nck = (r_eff + 15) >> 4;
    for (int c = 0; c < nck; ++c) {
      const uint4 u = __ldg(ex.U + ((size_t)rb * (ex.rs[0] >> 4) + c) * 32 + lane);
      const uint32_t af[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1 && !w.glue) break;
        if (16 * c >= ex.r[h]) continue;
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb) {
          const int col = gid + 8 * nb;
          const int rowc = row0 + (col < ncol ? col : 0);
          const float* tr = t + (size_t)rowc * w.t_ld + h * (w.t_ld / 2);
          const int rlim = w.row_rank ? min(ex.r[h], (int)w.row_rank[rowc * 3 + w.rank_slot0 + h]) : ex.r[h];
          uint32_t hi[2], lo[2];
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int rk = 16 * c + 2 * tig + 8 * hh;
            const float ta = (col < ncol && rk < rlim) ? tr[rk] : 0.f;
            const float tb = (col < ncol && rk + 1 < rlim) ? tr[rk + 1] : 0.f;
            t_hi_lo(ta, tb, hi[hh], lo[hh]);
          }
          mma16816(comp[h][nb], af, hi[0], hi[1]);
          mma16816(comp[h][nb], af, lo[0], lo[1]);
        }
      }
    }
    if (w.glue) {
      uint16_t* m = reinterpret_cast<uint16_t*>(out);
      const int ldm = w.n_rb * 8;
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 2 * tig + e + 8 * nb;
          if (col >= ncol) continue;
          const float up = tot[nb][e] + comp[0][nb][e];
          const float gt = tot[nb][e + 2] + comp[1][nb][e + 2];
          m[(size_t)(row0 + col) * ldm + rb * 8 + gid] = (uint16_t)f32_to_bf16_rn(up * (gt / (1.f + __expf(-gt))));
        }
    } else {
      float* o = reinterpret_cast<float*>(out);
      const int ldo = w.n_rb * kRows;
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = 2 * tig + (e & 1) + 8 * nb;
          if (col >= ncol) continue;
          o[(size_t)(row0 + col) * ldo + rb * kRows + gid + 8 * (e >> 1)] = tot[nb][e] + comp[0][nb][e];
        }
    }
    }
    if constexpr (KS) __syncthreads();                 // every warp, the same barrier: red is free again
  }
}

__global__ void moe_combine_kernel(const float* __restrict__ dout, int N, const float* __restrict__ gate, int T, int k,
                                   MoERoute rt, float* __restrict__ y) {
  asm volatile("griddepcontrol.wait;" ::: "memory");                 // PDL: the previous launch's outputs
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)T * N) return;
  const int tk = (int)(i / N), n = (int)(i % N);
  float acc = 0.f;
  for (int j = 0; j < k; ++j) {
    const int row = rt.tok_row[tk * k + j];
    if (row >= 0) acc = fmaf(gate[tk * k + j], dout[(size_t)row * N + n], acc);
  }
  y[i] = acc;
}

}  // namespace

// Programmatic dependent launch: every MoE kernel waits on the previous launch (griddepcontrol.wait)
// before reading its outputs, so only the launch latency and prologue overlap.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

cudaError_t moe_route(const int32_t* topk_idx, const float* topk_gate, int T, int k, int E, const MoERoute& rt,
                      const MoEDyn* dyn, cudaStream_t st) {
  if (T < 1 || T > 1024 || k < 1 || k > kMoEMaxK || E < 1 || E > 256) return cudaErrorInvalidValue;
  const size_t smem = (size_t)E * ((T + 31) / 32) * sizeof(unsigned);
  MoEDyn d{};
  if (dyn) d = *dyn;
  if (cudaError_t e = launch_pdl(moe_route_kernel, 1, kRouteThreads, smem, st, topk_idx, topk_gate, T, k, E, rt, d)) return e;
  return cudaGetLastError();
}

cudaError_t moe_prep(const uint16_t* x, int ldx, int K, int bits, int gather, const MoERoute& rt, int R_max,
                     uint16_t* xg, uint16_t* x16, float* xsig, cudaStream_t st) {
  const long long n = (long long)R_max * (K / 16);
  const unsigned grid = (unsigned)((n + 255) / 256);
  switch (bits) {
    case 2: if (cudaError_t e = launch_pdl(moe_prep_kernel<2>, grid, 256, 0, st, x, ldx, K, gather, rt, R_max, xg, x16, xsig)) return e; break;
    case 3: if (cudaError_t e = launch_pdl(moe_prep_kernel<3>, grid, 256, 0, st, x, ldx, K, gather, rt, R_max, xg, x16, xsig)) return e; break;
    case 4: if (cudaError_t e = launch_pdl(moe_prep_kernel<4>, grid, 256, 0, st, x, ldx, K, gather, rt, R_max, xg, x16, xsig)) return e; break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t moe_rank_proj(const MoEWin& w, const MoERoute& rt, int max_ent, const uint16_t* xg, float* t,
                          cudaStream_t st) {
  const int max_chunks = w.t_ld / 32;
  const long long jobs = (long long)max_ent * 2 * max_chunks;
  if (jobs == 0) return cudaSuccess;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (jobs < 2LL * sms) {
    if (cudaError_t e = launch_pdl(moe_rank_proj_kernel<16>, (unsigned)jobs, 16 * 32, 0, st, w, rt, max_ent, max_chunks, xg, t))
      return e;
  } else if (cudaError_t e = launch_pdl(moe_rank_proj_kernel<8>, (unsigned)jobs, 8 * 32, 0, st, w, rt, max_ent, max_chunks, xg, t)) {
    return e;
  }
  return cudaGetLastError();
}

cudaError_t moe_gemv(const MoEWin& w, int bits, const MoERoute& rt, int max_ent, const uint16_t* x16,
                     const float* xsig, const float* t, void* out, int max_cols, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long items = (long long)max_ent * w.n_rb;           // at most
  // few items (a handful of routed tokens): one item per CTA with K split over its kKSW warps
  const bool ks = items <= 8LL * sms;
  const long long need = ks ? items : (items + 3) / 4;
  const unsigned grid = (unsigned)(need < 16LL * sms ? need : 16LL * sms);
  const bool one = max_cols <= 8;                                  // NB8 = 1: at most 8 rows per entry
  cudaError_t e = cudaSuccess;
#define HC_MOE_LAUNCH(B_)                                                                                       \
  if (ks) {                                                                                                     \
    if (one) e = launch_pdl(moe_gemv_warp_kernel<B_, 1, true>, grid, kKSW * 32, 0, st, w, rt, x16, xsig, t, out);                \
    else     e = launch_pdl(moe_gemv_warp_kernel<B_, 2, true>, grid, kKSW * 32, 0, st, w, rt, x16, xsig, t, out);                \
  } else {                                                                                                      \
    if (one) e = launch_pdl(moe_gemv_warp_kernel<B_, 1, false>, grid, 128, 0, st, w, rt, x16, xsig, t, out);                      \
    else     e = launch_pdl(moe_gemv_warp_kernel<B_, 2, false>, grid, 128, 0, st, w, rt, x16, xsig, t, out);                      \
  }
  switch (bits) {
    case 2: HC_MOE_LAUNCH(2) break;
    case 3: HC_MOE_LAUNCH(3) break;
    case 4: HC_MOE_LAUNCH(4) break;
    default: return cudaErrorInvalidValue;
  }
#undef HC_MOE_LAUNCH
  return e;
}

cudaError_t moe_combine(const float* dout, int N, const float* topk_gate, int T, int k, const MoERoute& rt,
                        float* y, cudaStream_t st) {
  const long long n = (long long)T * N;
  if (cudaError_t e = launch_pdl(moe_combine_kernel, (unsigned)((n + 255) / 256), 256, 0, st, dout, N, topk_gate, T, k, rt, y)) return e;
  return cudaGetLastError();
}

}  // namespace hc
