// Fused decode kernel: one launch evaluates a whole compensation window
//
//     y[b, n] = Σ_g s[n,g] · Σ_{k∈g} (q[n,k] − z[n,g]) · x[b,k]  +  Σ_{j<r} U[n,j] · t[b,j],
//     t[b, j] = Σ_k V[j,k] · x[b,k]                                      (north_star)
//
// Design (DESIGN.md §"Decode kernel"):
//  * one CTA work item is a row block (16 output rows × all of K), striped over a grid of one
//    resident wave (persistent loop beyond that); the rank projection is spread over every tile warp
//    of the grid as a small prologue;
//  * each warp streams its tiles — a (row-block, group) record or a 1 KB V piece — from HBM with
//    cp.async.bulk (TMA engine, L2 evict-first) into a private 4-slot shared-memory ring guarded
//    by mbarriers; W is never materialised;
//  * PDL: weight tiles (and U fragments) are requested before griddepcontrol.wait, i.e. while the
//    previous kernel in the stream is still finishing; x, t, y and the counters are touched only
//    after it;
//  * x is staged once per CTA in shared memory (rows padded so 128-bit fragment loads are
//    bank-conflict-free), or read through L1 when it does not fit;
//  * codes -> fp16 A-fragments with at most one shift per word + one lop3 per register (the 0x6400
//    magic, exact integers), minus the per-group zero with one hsub2 (exact), times x' = x·2^-fp
//    (fp16, exact) on mma.sync m16n8k16 with fp32 accumulation; per-group partials are scaled by the
//    fp32 group scale afterwards;
//  * the 8 warps' partial sums are reduced in shared memory in a fixed order; the CTA's epilogue
//    warp adds U[:, :r]·t with t split into bf16 hi + lo (fp32-accurate) on the same mma and
//    writes y once (fp32, or bf16 = RNE of the fp32 value), optionally adding a bf16 residual;
//  * t is produced inside the launch with tiered 64-bit fixed-point atomics (tacc_add: one atomic per
//    fp32 partial, rounded once to 24+ bits; integer adds are associative, so t is deterministic); epilogues
//    acquire a release counter.  The accumulators and counters self-reset before the kernel exits.
//  * fp16 path: the B operand carries a per-(group, batch row) power-of-two prescale when a group's
//    range needs it (R20), so any bf16 x is accepted.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <type_traits>

#include "decode.h"
#include "options.h"
#include "decode_dev.cuh"
#include "layout.h"

namespace hc {
__device__ unsigned long long* g_dtrace = nullptr;   // dev tracing (HC_DEC_TRACE builds)
}
#include "decode_i8.cuh"

namespace hc {

#ifndef HC_POLL_RELAXED
#define HC_POLL_RELAXED 0
#endif
#ifndef HC_DEP_SLEEP
#define HC_DEP_SLEEP 64   // ns between polls of the producer window's counter
#endif
#ifndef HC_DEC_TRACE
#define HC_DEC_TRACE 0
#endif
// dev tracing: globaltimer stamps per (launch slot, CTA): [0] start, [1] after the PDL wait (epilogue),
// [2] first FULL passed, [3] last FULL passed, [4] epilogue done, [5] t ready
__device__ __forceinline__ void dtrace(const DArgs& a, int ev) {
#if HC_DEC_TRACE
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (g_dtrace) g_dtrace[((size_t)a.trace_slot * 512 + blockIdx.x) * 16 + ev] = t;
#endif
}
// Peer mode, end of the stack: wait for every rank's rows of the last window, copy them out, reset the counter.
__global__ void peer_wait_copy_kernel(const unsigned* cnt, unsigned target, unsigned* reset, const uint16_t* src,
                                      uint16_t* out, size_t n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) wait_sys(cnt, target);
  __syncthreads();
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) out[i] = __ldcg(src + i);
  __syncthreads();
  if (threadIdx.x == 0 && reset) *reset = 0u;
}

cudaError_t launch_peer_wait_copy(const unsigned* cnt, unsigned target, unsigned* reset, const uint16_t* src, uint16_t* out,
                                  size_t n_elems, cudaStream_t st) {
  peer_wait_copy_kernel<<<1, 1024, 0, st>>>(cnt, target, reset, src, out, n_elems);
  return cudaGetLastError();
}

cudaError_t decode_set_trace(void* buf) { return cudaMemcpyToSymbol(g_dtrace, &buf, sizeof(buf)); }


// Warp roles: warps 0..7 stream and contract tiles; warps 8 (.. 8 + epi - 1) are the epilogue warps (reduction of
// the 8 partial sums, U·t, output; item k of a CTA -> epilogue warp k % epi, dec_epi_warps); the last warp issues
// the TMA ring.  Named barriers hand the shared reduction buffer red[s] (s = k % kRedSlots) between them:
//   FULL[s]  (red_full_id): 256 tile threads arrive, the item's epilogue warp syncs
//   EMPTY[s] (red_empty_id): that epilogue warp arrives after reading red[s], the tile warps sync before
//                            writing red[s] again kRedSlots items later.
// Rank projection t = V·x: every tile warp of the grid first contracts an equal share of the
// window's 1 KB V pieces (requested before its weight tiles) and adds its partial into the
// window's t accumulators with 64-bit fixed-point atomics (exact integer adds: t is bit-identical
// for any arrival order), then bumps v_done; each CTA's epilogue warp acquires v_done once and reads
// t while its tile warps are still streaming.
// Wait for this window's inputs: the producer window's completion counter (acquire; every warp that
// reads activations calls this), else the programmatic-dependent-launch grid dependency.
__device__ __forceinline__ void dep_wait(const DArgs& a, int lane) {
  if (a.dep_cnt) {
    if (a.npeer > 1) {                                            // peer mode: every rank's producer adds into it
      if (lane == 0) {
        wait_sys(a.dep_cnt, a.dep_target);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      __syncwarp();
      return;
    }
    if (lane == 0) {
#if HC_POLL_RELAXED
      while (ld_relaxed(a.dep_cnt) < a.dep_target) __nanosleep(HC_DEP_SLEEP);
      (void)ld_acquire(a.dep_cnt);   // (a fence.acq_rel here measured slower than the second load)
#else
      // acquire loads in the poll: the load that sees the target is the acquire (one L2 round trip less
      // than relaxed polling + a separate acquire; ~1-2 µs under a full weight stream)
      while (ld_acquire(a.dep_cnt) < a.dep_target) __nanosleep(HC_DEP_SLEEP);
#endif
      asm volatile("fence.proxy.async.global;" ::: "memory");   // generic writes -> async-proxy (TMA) reads
    }
    __syncwarp();
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
}

// L2 prefetch of this CTA's share of the next window's records (DArgs::pf_items); lane j of nl lanes takes
// the CTA's next-window items j, j + nl, ...
__device__ __forceinline__ void prefetch_next_window(const DArgs& a, int j, int nl) {
  if (a.pf_items <= 0) return;
  const int total = a.pf_rb_end[a.pf_nm - 1];
  for (; j < a.pf_items; j += nl) {
    const int it = blockIdx.x + j * gridDim.x;
    if (it >= total) return;
    int i = 0, b0 = 0;
#pragma unroll
    for (int q = 0; q < kMaxMembers - 1; ++q)
      if (q + 1 < a.pf_nm && it >= a.pf_rb_end[q]) { i = q + 1; b0 = a.pf_rb_end[q]; }
    prefetch_l2(a.pf_rec[i] + (size_t)(it - b0) * a.pf_item_bytes, a.pf_item_bytes);
  }
}

// I8: int8 tensor-core path (decode_i8.cuh; BITS = 4, NB8 = 1, B <= 2): x staged as x8 digits
template <int BITS, int NB8, bool XS, bool I8, bool F8>
__global__ void __launch_bounds__(dec_block(I8), HC_DEC_MINB) decode_kernel(const __grid_constant__ DArgs a) {
  constexpr int kEpiWarps = dec_epi_warps(I8);
  constexpr int kProdWarp = kDecodeWarps + kEpiWarps;       // the producer (TMA issue) warp
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  constexpr int kBlk = kTPB * kTileMax;
  // records per bulk-copy block: as many as the block holds (2-bit records are half the size)
  constexpr int kRPB = (kBlk / rec_bytes(BITS)) < 1 ? 1 : (kBlk / rec_bytes(BITS));
  float* red = reinterpret_cast<float*>(smem + (size_t)kDecodeWarps * kNBuf * kBlk);        // [kRedSlots][8][32][4·NB8]
  uint4* ubuf = reinterpret_cast<uint4*>(red + kRedSlots * kDecodeWarps * 32 * 4 * NB8);     // [2][kUPre][32]
  uint64_t* bars_all = reinterpret_cast<uint64_t*>(ubuf + 2 * kUPre * 32);
  uint64_t* ubar = bars_all + kDecodeWarps * kNBuf;       // [2]
  uint64_t* xbar = ubar + 2;
  uint64_t* fbar = xbar + 1;                              // t forwarding: Vn blocks landed, buffer 0
  uint64_t* fbar1 = xbar + 3;                             //   ... buffer 1 (the Vn blocks are double-buffered)
  uint64_t* dbar = xbar + 2;                              // dataflow dependency met (epilogue -> tile warps)
  uint64_t* ebars_all = xbar + 4;                         // [8 warps][kNBuf] ring slot consumed (empty; +1 pad: tsm 16-B aligned)
  uint64_t* e2bar = ebars_all + kDecodeWarps * kNBuf;    // [2]: [0] epilogue warp 0 passed the dependency wait (+1 pad)
  // t fragments: one copy per epilogue warp, each loads t itself (measured: sharing one copy, the first warp to
  // need t loading it for both, C2 635 -> 578 tokens/s, C1 1127 -> 846 GB/s)
  uint4* tsm_all = reinterpret_cast<uint4*>(e2bar + 2);  // [epi warp][n_chunks][NB8][32] t hi|lo fragments
  uint16_t* xt_all = reinterpret_cast<uint16_t*>(tsm_all + (size_t)kEpiWarps * a.n_chunks * NB8 * 32);   // [epi warp][16 k][16 cols]
  uint4* fbuf = reinterpret_cast<uint4*>(xt_all + 256 * kEpiWarps);                  // [2][fwd_chunks][32] Vn fragments
  unsigned* misc = reinterpret_cast<unsigned*>(fbuf + (size_t)(a.fwd ? a.fwd_chunks : 0) * 64);   // [4]: [0] XS σ any, [1] x' slow path, [2] epilogue warp 1 row blocks
  float* fsg = reinterpret_cast<float*>(misc + 4);                                   // XS: 2^σ [G][B]
  uint16_t* xs = reinterpret_cast<uint16_t*>(fsg + ((XS && !I8) ? ((a.G * a.B + 3) & ~3) : 0));
  const int xs_ld = a.K + 32;   // +64 B per row: consecutive batch rows fall in disjoint banks

  if (lane == 0) {
    if (warp < kDecodeWarps) {
#pragma unroll
      for (int s = 0; s < kNBuf; ++s) {
        mbar_init(&bars_all[warp * kNBuf + s], 1);
        mbar_init(&ebars_all[warp * kNBuf + s], 32);
      }
    } else if (warp == kDecodeWarps) {   // epilogue warp 0
      mbar_init(&ubar[0], 1); mbar_init(&ubar[1], 1); mbar_init(xbar, 1); mbar_init(fbar, 1); mbar_init(dbar, 1);
      mbar_init(fbar1, 1);
      mbar_init(e2bar, 1);
      misc[0] = 0u; misc[1] = 0u; misc[2] = 0u;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const int n_items = a.n_rb;
  // the V·x share lives on the first CTAs (started first), ~kVPerWarp 1 KB pieces per tile warp
  const int n_vp = a.t_in ? 0 : a.n_chunks * (F8 ? 2 : 4) * a.G;   // t_in: t accumulated by the producer of x
  const int n_vctas = n_vp == 0 ? 0 : min((int)gridDim.x, (n_vp + kDecodeWarps * kVPerWarp - 1) / (kDecodeWarps * kVPerWarp));
  const int n_vwarps = n_vctas * kDecodeWarps;            // v_done target

  if (warp == kProdWarp) {
    // ======================= producer warp =======================
    // Lane w issues tile warp w's ring: its V pieces, then blocks of up to kRPB consecutive records of
    // each row-block share (warp_share), each into the next slot once the tile warp released it
    // (empty mbarrier).  Nothing here reads activations, so it never waits on the producer window:
    // a window's weight stream starts while the previous window is finishing.
    if (lane < kDecodeWarps) {
      const int w = lane;
      uint8_t* wbufs = smem + (size_t)w * kNBuf * kBlk;
      uint64_t* wfull = bars_all + w * kNBuf;
      uint64_t* wempty = ebars_all + w * kNBuf;
      const uint64_t pol_w = evict_first_policy();
      const int gw = blockIdx.x * kDecodeWarps + w;
      const bool v_w = gw < n_vwarps;
      int vp = v_w ? (int)((long long)gw * n_vp / n_vwarps) : 0;
      const int vp_end = v_w ? (int)((long long)(gw + 1) * n_vp / n_vwarps) : 0;
      int p_item = blockIdx.x, p_t = 0;
      Share sh = p_item < n_items ? warp_share<BITS>(a, p_item, w) : Share{nullptr, 0, 1024, 0, 0, 0};
      int slot = 0;
      uint32_t round = 0;
      while (true) {
        const uint8_t* src;
        uint32_t bytes;
        if (vp < vp_end) {
          int g, part;
          src = F8 ? v_piece8(a, vp, g, part) : v_piece(a, vp, g, part);
          bytes = 1024u;
          ++vp;
        } else {
          while (p_item < n_items && p_t >= sh.n) {
            p_item += gridDim.x;
            p_t = 0;
            if (p_item < n_items) sh = warp_share<BITS>(a, p_item, w);
          }
          if (p_item >= n_items) break;
          const int nt = min(kRPB, sh.n - p_t);
          src = sh.base + (size_t)p_t * sh.tb;
          bytes = (uint32_t)(nt * sh.tb);
          p_t += nt;
        }
        if (round > 0)
          while (!mbar_try_wait(&wempty[slot], (round - 1) & 1u)) {}
        mbar_expect_tx(&wfull[slot], bytes);
        bulk_copy(wbufs + slot * kBlk, src, bytes, &wfull[slot], pol_w);
        if (++slot == kNBuf) { slot = 0; ++round; }
      }
      if (!a.pf_at_start) prefetch_next_window(a, lane, kDecodeWarps);
    } else if (a.pf_at_start) {
      prefetch_next_window(a, lane - kDecodeWarps, 32 - kDecodeWarps);
    }
    return;
  }

  if (warp >= kDecodeWarps) {
    // ======================= epilogue warps =======================
    // warp e takes the CTA's items k = e, e + kEpiWarps, ... (item parity = reduction buffer = e when 2 warps)
    const int e_w = warp - kDecodeWarps;
    uint4* tsm = tsm_all + (size_t)e_w * a.n_chunks * NB8 * 32;
    uint16_t* xt = xt_all + 256 * e_w;
    if (lane == 0 && e_w == 0) dtrace(a, 0);
    auto prefetch_u = [&](int rb, int par) {   // U fragments of a row-block item -> ubuf[par]
      if (rb >= n_items) return;
      const DMember& m = a.m[member_of_rb(a, rb)];
      const int r_eff = a.glue ? max(a.m[0].r, a.m[1].r) : m.r;
      const int nck = min((r_eff + 15) >> 4, kUPre);
      if (nck == 0) return;
      if (lane == 0) {
        const uint32_t cb = F8 ? 256u : 512u;          // bytes of one rank chunk of a row block's U fragments
        const uint32_t bytes = (uint32_t)nck * cb;
        mbar_expect_tx(&ubar[par], bytes);
        bulk_copy(ubuf + par * kUPre * 32,
                  reinterpret_cast<const uint8_t*>(m.U) + (size_t)(rb - m.rb_begin) * (m.r_stored >> 4) * cb, bytes,
                  &ubar[par], evict_first_policy());
      }
    };
    // t forwarding: the next window's natural-k V fragments of an item's 16-k output block -> fbuf[buf]
    // (double-buffered: the first item's before the dependency wait, then one item ahead; weights only)
    auto prefetch_fwd = [&](int it, int buf) {
      if (!a.fwd || it >= n_items || lane != 0) return;
      const DMember& mm = a.m[member_of_rb(a, it)];
      const int n0 = (a.npeer > 1 ? mm.full_off : mm.row_off) + (it - mm.rb_begin) * (a.glue ? 8 : kRows);
      if (n0 < a.fwd_lo || n0 >= a.fwd_hi) return;
      const int kb = (n0 - a.fwd_lo) >> 4;
      uint64_t* fb = buf ? fbar1 : fbar;
      mbar_expect_tx(fb, (uint32_t)a.fwd_chunks * 512u);
      for (int i = 0; i < a.fwd_nm; ++i) {
        const int nc = a.fwd_cb[i + 1] - a.fwd_cb[i];
        if (nc > 0)
          bulk_copy(fbuf + ((size_t)buf * a.fwd_chunks + a.fwd_cb[i]) * 32, a.fwd_vn[i] + (size_t)kb * a.fwd_rs[i] * 32,
                    (uint32_t)nc * 512u, fb, evict_first_policy());
      }
    };
    // warm the SM's constant cache with every line of the kernel parameters (the member table is indexed
    // dynamically on the t / epilogue critical path; a constant-cache miss there costs an L2 round trip under
    // the weight stream), while the window still waits for its producer
    if (lane * 64 < (int)sizeof(DArgs)) {
      const uint32_t v = reinterpret_cast<const uint32_t*>(&a)[lane * 16];
      asm volatile("" ::"r"(v));
    }
    const int item0 = blockIdx.x + e_w * (int)gridDim.x;
    prefetch_u(item0, e_w);                              // weights: before the PDL wait
    prefetch_fwd(item0, e_w);
    // dependency: warp 0 acquires the producer's counter (or waits on the grid dependency); the other epilogue
    // warp waits on warp 0's mbarrier arrive (cumulative, like the tile warps' dbar) instead of polling the
    // producer's counter a second time
    if (e_w == 0) {
      dep_wait(a, lane);
      if (kEpiWarps > 1 && a.dep_cnt && lane == 0) mbar_arrive(e2bar);
    } else if (!a.dep_cnt) {
      dep_wait(a, lane);
    } else {
      while (!mbar_try_wait(e2bar, 0)) {}
    }
    if (e_w == 0 && blockIdx.x == 0 && a.clr_max)        // the max buffer the next window publishes into (R20)
      for (int i = lane; i < a.clr_n; i += 32) a.clr_max[i] = 0u;
    // release the tile warps: one mbarrier arrive after the acquire (cumulative through the mbarrier's
    // release / acquire); the tile warps read activations only after their wait on it
    if ((!XS || I8) && a.dep_cnt && lane == 0 && e_w == 0) mbar_arrive(dbar);
    if (lane == 0 && e_w == 0) dtrace(a, 1);
    if constexpr (XS && !I8) {
      if (lane == 0 && e_w == 0) {
        mbar_expect_tx(xbar, (uint32_t)(a.B * a.K * 2));
        for (int b = 0; b < a.B; ++b)
          bulk_copy(xs + (size_t)b * xs_ld, a.x + (size_t)b * a.ldx, (uint32_t)(a.K * 2), xbar, evict_last_policy());
      }
    }
    unsigned u_phase = 0;   // bit p = phase of ubar[p]
    unsigned f_phase = 0;
    bool t_ready = false;
    bool t_deep = false;   // the extra-tier flag of this window's t (read with t; reset on the exit path)
    int my_rb = 0;
    int k = e_w;
    for (int item = item0; item < n_items; item += kEpiWarps * (int)gridDim.x, k += kEpiWarps) {
      const int par = k & 1;
      const DMember& m = a.m[member_of_rb(a, item)];
      const int r_eff = a.glue ? max(a.m[0].r, a.m[1].r) : m.r;
      if (!t_ready && r_eff > 0) {
        // once per CTA, while the tile warps still stream: acquire t (all tile warps of the grid
        // have added their V·x shares) and keep its fragments in smem (each epilogue warp its own copy)
        unsigned seen = 0;
        if (lane == 0 && n_vctas > 0) {                 // t_in: ordered by the dependency wait already
#if HC_POLL_RELAXED
          while (ld_relaxed(&a.cnt[0]) < (unsigned)n_vctas) __nanosleep(32);
          seen = ld_acquire(&a.cnt[0]);
#else
          while ((seen = ld_acquire(&a.cnt[0])) < (unsigned)n_vctas) __nanosleep(32);
#endif
          if (e_w == 0) dtrace(a, 11);                   // v_done observed
        }
        // the t loads below are plain (non-volatile) asm so that they batch: their addresses carry a data
        // dependency on the acquired counter value so the compiler cannot move them above the acquire
        __syncwarp();                                    // orders every lane's t loads after lane 0's acquire
        const long long* tq = a.tacc + zero_dep(__shfl_sync(0xFFFFFFFFu, seen, 0));
        // t as bf16 hi + lo B-fragments of the U·t mma (fp32-accurate), ranks >= r masked to 0.  Tier 0 here, each
        // lane loading the words of its own fragments (R22); the extra-tier flag is loaded first and consumed after
        // the loop.  No branch may sit between the loads of this loop (a branch inside the unrolled loop
        // serialises them into one L2 round trip per chunk: +2.5 µs on C1).
        t_deep = __ldcg(a.tacc + (size_t)kTCopies * a.n_chunks * kTChunk) != 0;
        // (the loop is unrolled by the chunk count's bucket: measured C2 +2.6% at 8 chunks in flight for windows
        // with > 4 chunks, C1 (4 chunks) -4% with the unroll-8 loop)
        auto tier0 = [&](auto unroll_c) {
          constexpr int kU = decltype(unroll_c)::value;
#pragma unroll kU
          for (int cc = 0; cc < a.n_chunks; ++cc) {
            const DMember& mt = a.m[member_of_chunk(a, cc)];
            const int r0 = 16 * (cc - mt.chunk_begin) + 2 * tig;
#pragma unroll
            for (int nb = 0; nb < NB8; ++nb) {
              const long long* src = a.tacc + (size_t)cc * kTChunk + ((gid + 8 * nb) & 15) * 16 + 2 * tig;
              // only the lanes of batch columns < B load (the others' words are zero): predicated, not branched
              const bool on = gid + 8 * nb < a.B;
              const long long tr[4] = {ldcg_if(src, on), ldcg_if(src + 1, on), ldcg_if(src + 8, on), ldcg_if(src + 9, on)};
              uint32_t hi[2], lo[2];
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                float ta = (r0 + 8 * hh < mt.r) ? (float)tr[2 * hh] * 0x1p-36f : 0.f;
                float tb = (r0 + 8 * hh + 1 < mt.r) ? (float)tr[2 * hh + 1] * 0x1p-36f : 0.f;
                if constexpr (F8) {                        // t'_j = u_scale_j·t_j (unconditional, in-range loads)
                  ta *= mt.us[min(r0 + 8 * hh, mt.r_stored - 1)];
                  tb *= mt.us[min(r0 + 8 * hh + 1, mt.r_stored - 1)];
                }
                t_hi_lo(ta, tb, hi[hh], lo[hh]);
              }
              tsm[((size_t)cc * NB8 + nb) * 32 + lane] = make_uint4(hi[0], hi[1], lo[0], lo[1]);
            }
          }
        };
        if (a.n_chunks > 4) tier0(std::integral_constant<int, 8>{});
        else tier0(std::integral_constant<int, 4>{});
        if (lane == 0 && e_w == 0) dtrace(a, 13);
        // rare (outlier or tiny activations, R22): every tier, all loads of the pass in flight together
        if (t_deep) {
          t_fragments_deep_load<NB8>(a, tq, tsm, lane);
          t_fragments_build<NB8>(a, tsm, lane);
        }
        if (lane == 0 && e_w == 0) dtrace(a, 14);
        __syncwarp();
        t_ready = true;
        if (lane == 0 && e_w == 0) dtrace(a, 5);
      }
      // t forwarding: this item's outputs are x of the next window at k = n0 - fwd_lo .. (16 or 8 of them);
      // fetch the next window's natural-k V fragments of that 16-k block while the tile warps work
      // first output column of this item: in the window output (local), or in the full gathered output (peer
      // mode: the column the other ranks and the next window see)
      const int oc0 = (a.npeer > 1 ? m.full_off : m.row_off) + (item - m.rb_begin) * (a.glue ? 8 : kRows);
      const int f_n0 = oc0;
      const bool f_on = a.fwd && f_n0 >= a.fwd_lo && f_n0 < a.fwd_hi;
      if (kEpiWarps == 1) prefetch_fwd(item + (int)gridDim.x, (k + 1) & 1);   // the next item's Vn block (this one's is in flight)
      // ---- independent of the tile warps (so done before waiting for their partial sums): U[:, :r]·t
      // (U prefetched one item ahead) and the residual (its producer window is >= 2 windows back,
      // complete once this window's dependency was met)
      const int rbl = item - m.rb_begin;
      // U·t: plain windows use the member's own chunks for all 16 rows; a fused SiLU window runs
      // the up chunks (rows 0-7 = up rows) and the gate chunks (rows 8-15 = gate rows) separately
      float comp[2][NB8][4];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) comp[h][nb][e] = 0.f;
      if (r_eff > 0) {
        const int nck = (r_eff + 15) >> 4;
        while (!mbar_try_wait(&ubar[par], (u_phase >> par) & 1u)) {}
        u_phase ^= 1u << par;
        for (int c = 0; c < nck; ++c) {
          uint32_t af[4];
          if constexpr (F8) {                            // e4m3 fragments, converted exactly (t carries u_scale)
            const uint2 u8 = (c < kUPre) ? reinterpret_cast<const uint2*>(ubuf + par * kUPre * 32)[c * 32 + lane]
                                         : __ldg(reinterpret_cast<const uint2*>(m.U) + ((size_t)rbl * (m.r_stored >> 4) + c) * 32 + lane);
            e4m3x8_frag(u8, af);
          } else {
            const uint4 u = (c < kUPre) ? ubuf[(par * kUPre + c) * 32 + lane]
                                        : __ldg(m.U + ((size_t)rbl * (m.r_stored >> 4) + c) * 32 + lane);
            af[0] = u.x; af[1] = u.y; af[2] = u.z; af[3] = u.w;
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !a.glue) break;
            const DMember& mt = a.glue ? a.m[h] : m;      // whose rank space / t
            if (16 * c >= mt.r) continue;
#pragma unroll
            for (int nb = 0; nb < NB8; ++nb) {
              const uint4 q = tsm[((size_t)(mt.chunk_begin + c) * NB8 + nb) * 32 + lane];
              mma16816(comp[h][nb], af, q.x, q.y);     // U·t_hi
              mma16816(comp[h][nb], af, q.z, q.w);     // U·t_lo
            }
          }
        }
      }
      float res[NB8][4];
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          res[nb][e] = 0.f;
          const int b = 2 * tig + (e & 1) + 8 * nb;
          if (a.resid && !a.glue && b < a.B)
            res[nb][e] = bf16_bits_to_f32(__ldcg(a.resid + (size_t)b * a.ld_resid + oc0 + gid + 8 * (e >> 1)));
        }
      if (f_on) {                                        // zero the x tile (cols >= B and the other 8 k stay 0)
        reinterpret_cast<uint4*>(xt)[lane] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
      }
      const int rs = k % kRedSlots;                      // reduction slot of this item
      asm volatile("bar.sync %0, %1;" ::"r"(red_full_id(rs)), "n"(kDecodeThreads) : "memory");   // FULL[rs]
      if (lane == 0) { if (k == 0) dtrace(a, 2); if (item + (int)gridDim.x >= n_items) dtrace(a, 3); }
      float fin[NB8][4];
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) fin[nb][e] = 0.f;
#pragma unroll
      for (int w = 0; w < kDecodeWarps; ++w) {            // fixed order: deterministic
        const float* src = red + ((size_t)(rs * kDecodeWarps + w) * 32 + lane) * 4 * NB8;
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb) {
          const float4 v = *reinterpret_cast<const float4*>(src + 4 * nb);
          fin[nb][0] += v.x; fin[nb][1] += v.y; fin[nb][2] += v.z; fin[nb][3] += v.w;
        }
      }
      if (item + kRedSlots * (int)gridDim.x < n_items)
        asm volatile("bar.arrive %0, %1;" ::"r"(red_empty_id(rs)), "n"(kDecodeThreads) : "memory");   // EMPTY[rs]
      if (kEpiWarps == 1) prefetch_u(item + gridDim.x, par ^ 1);
      else prefetch_u(item + kEpiWarps * (int)gridDim.x, par);   // this warp's next item (its U·t is done)

      uint32_t xm[NB8][2];                               // largest |bf16 y| per batch row (x' range, R20)
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb) xm[nb][0] = xm[nb][1] = 0u;
      if (a.glue) {
        // m[b][8·rbl + gid] = silu(gate) · up, gate = row gid+8 (c2, c3), up = row gid (c0, c1)
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int b = 2 * tig + e + 8 * nb;
            if (b >= a.B) continue;
            const float up = fin[nb][e] + comp[0][nb][e];
            const float gt = fin[nb][e + 2] + comp[1][nb][e + 2];
            const float v = up * (gt / (1.f + __expf(-gt)));
            const int n = m.row_off + rbl * 8 + gid;
            if (a.y_bf16) {
              const uint16_t bits = (uint16_t)f32_to_bf16_rn(v);
              if (a.npeer > 1) {
#pragma unroll 1
                for (int q = 0; q < a.npeer; ++q) a.ypeer[q][(size_t)b * a.ld_full + oc0 + gid] = bits;
              } else {
                reinterpret_cast<uint16_t*>(a.y)[(size_t)b * a.ldy + n] = bits;
              }
              if (f_on) xt[(((f_n0 - a.fwd_lo) & 15) + gid) * 16 + b] = bits;
              if (a.y16 && n >= a.y16_lo && n < a.y16_hi) write_xprime<BITS>(a, b, n, bits);
              xm[nb][e] = max(xm[nb][e], (uint32_t)bits & 0x7FFFu);
            } else {
              reinterpret_cast<float*>(a.y)[(size_t)b * a.ldy + n] = v;
            }
          }
      } else {
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int b = 2 * tig + (e & 1) + 8 * nb;
            if (b >= a.B) continue;
            const int n = m.row_off + rbl * kRows + gid + 8 * (e >> 1);
            const float v = fin[nb][e] + comp[0][nb][e] + res[nb][e];
            if (a.y_bf16) {
              const uint16_t bits = (uint16_t)f32_to_bf16_rn(v);
              if (a.npeer > 1) {
#pragma unroll 1
                for (int q = 0; q < a.npeer; ++q) a.ypeer[q][(size_t)b * a.ld_full + oc0 + gid + 8 * (e >> 1)] = bits;
              } else {
                reinterpret_cast<uint16_t*>(a.y)[(size_t)b * a.ldy + n] = bits;
              }
              if (f_on) xt[(gid + 8 * (e >> 1)) * 16 + b] = bits;
              if (a.y16 && n >= a.y16_lo && n < a.y16_hi) write_xprime<BITS>(a, b, n, bits);
              xm[nb][e & 1] = max(xm[nb][e & 1], (uint32_t)bits & 0x7FFFu);
            } else {
              reinterpret_cast<float*>(a.y)[(size_t)b * a.ldy + n] = v;
            }
          }
      }
      if (a.y16 && a.y16_max && f_n0 >= a.y16_lo && f_n0 < a.y16_hi) publish_xmax<NB8>(a, f_n0, xm, lane);
      if (f_on) {
        // t_next[c][col][rank] += Σ_{k in this block} Vn[c][rank][k] · x[col][k]  (bf16 mma, fp32, then
        // 2^-28 fixed point: integer adds, so the sum is independent of the order items arrive)
        __syncwarp();
        uint32_t b0[NB8], b1[NB8];
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb) {
          const int col = gid + 8 * nb;
          b0[nb] = (uint32_t)xt[(2 * tig) * 16 + col] | ((uint32_t)xt[(2 * tig + 1) * 16 + col] << 16);
          b1[nb] = (uint32_t)xt[(2 * tig + 8) * 16 + col] | ((uint32_t)xt[(2 * tig + 9) * 16 + col] << 16);
        }
        const int fb = k & 1;
        while (!mbar_try_wait(fb ? fbar1 : fbar, (f_phase >> fb) & 1u)) {}
        f_phase ^= 1u << fb;
        const uint4* fbk = fbuf + (size_t)fb * a.fwd_chunks * 32;
#pragma unroll 4
        for (int cc = 0; cc < a.fwd_chunks; ++cc) {
          const uint4 v4 = fbk[cc * 32 + lane];
          const uint32_t af[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
          for (int nb = 0; nb < NB8; ++nb) {
            float tp[4] = {0.f, 0.f, 0.f, 0.f};
            mma16816(tp, af, b0[nb], b1[nb]);
            if (NB8 == 1 && a.B <= 2) {
              // B <= 2: the 16·B valid partials sit in the tig = 0 lanes; gather them one per lane so the
              // fixed-point adds run as one warp-wide sequence instead of four predicated ones
              const int rk = lane & 15, cl = lane >> 4;                  // lane -> (rank, batch column)
              const int src = 4 * (rk & 7), e0 = 2 * (rk >> 3);
              const float v0 = __shfl_sync(0xFFFFFFFFu, tp[0], src), v1 = __shfl_sync(0xFFFFFFFFu, tp[1], src);
              const float v2 = __shfl_sync(0xFFFFFFFFu, tp[2], src), v3 = __shfl_sync(0xFFFFFFFFu, tp[3], src);
              const float v = e0 == 0 ? (cl ? v1 : v0) : (cl ? v3 : v2);
              if (cl < a.B) {
                if (a.npeer > 1) {
#pragma unroll 1
                  for (int q = 0; q < a.npeer; ++q) tacc_add(a.fwdpeer[q], a.fwd_chunks, cc, cl, rk, v);
                } else {
                  tacc_add(a.fwd_tacc, a.fwd_chunks, cc, cl, rk, v);
                }
              }
              continue;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int col = 2 * tig + (e & 1) + 8 * nb, rank = gid + 8 * (e >> 1);
              if (col < a.B) {
                if (a.npeer > 1) {                                 // partial-t exchange: this rank's slice, every rank
#pragma unroll 1
                  for (int q = 0; q < a.npeer; ++q) tacc_add(a.fwdpeer[q], a.fwd_chunks, cc, col, rank, tp[e]);
                } else {
                  tacc_add(a.fwd_tacc, a.fwd_chunks, cc, col, rank, tp[e]);
                }
              }
            }
          }
        }
        __syncwarp();                                    // fbuf / xt reused by the next item
      }
      if (kEpiWarps > 1) prefetch_fwd(item + kEpiWarps * (int)gridDim.x, par);   // this warp's buffer is free again
      ++my_rb;
    }
    if (lane == 0 && e_w == 0) dtrace(a, 4);
    // one counter update per CTA: the CTA completing the last row block resets t and the counters
    // (every t reader is a row-block epilogue, all of which have finished by then)
    __syncwarp();
    if constexpr (kEpiWarps > 1) {
      // the epilogue warps meet (named barrier 6); warp 0 publishes the CTA's row blocks (cumulativity through
      // the barrier orders warp 1's output stores before warp 0's release)
      if (e_w == 1 && lane == 0) misc[2] = (unsigned)my_rb;
      asm volatile("bar.sync 6, %0;" ::"n"(kEpiWarps * 32) : "memory");
      if (e_w != 0) return;
      my_rb += (int)misc[2];
    }
    unsigned last = 0;
    if (lane == 0 && my_rb > 0) {
      const unsigned old = add_acq_rel(&a.cnt[1], (unsigned)my_rb);
      last = (old + (unsigned)my_rb == (unsigned)a.n_rb);
      if (a.npeer > 1)                                     // peer mode: this CTA's rows of the gather, on every rank
        for (int q = 0; q < a.npeer; ++q) red_release_sys(a.dpeer[q], (unsigned)my_rb);
    }
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      // the flag as read with t (a CTA that never read t loads it here)
      const bool xt = t_ready ? t_deep : (__ldcg(a.tacc + (size_t)kTCopies * a.n_chunks * kTChunk) != 0);
      tacc_reset(a.tacc, a.n_chunks, a.B, xt, lane);
      if (lane == 0) {
        a.cnt[0] = 0u;
        if (!a.keep_done) a.cnt[1] = 0u;             // else the consumer window resets it
        if (a.dep_reset) *a.dep_reset = 0u;          // every CTA of this window passed its wait
      }
    }
    return;
  }

  // ======================= tile warps =======================
  uint8_t* bufs = smem + (size_t)warp * kNBuf * kBlk;    // [kNBuf][kBlk], filled by the producer warp
  uint64_t* bars = bars_all + warp * kNBuf;
  uint64_t* ebars = ebars_all + warp * kNBuf;
  // this warp's share of the window's V pieces (rank projection)
  const int gw = blockIdx.x * kDecodeWarps + warp;
  const bool v_warp = gw < n_vwarps;
  const int vp0 = v_warp ? (int)((long long)gw * n_vp / n_vwarps) : 0;
  const int vp1 = v_warp ? (int)((long long)(gw + 1) * n_vp / n_vwarps) : 0;
  // tile warps read activations only through the x staged by the epilogue warp (XS, ordered by its
  // acquire and the x mbarrier), except for V pieces and unstaged x: only then do they wait themselves
  if (!a.dep_cnt) dep_wait(a, lane);
  else if (!XS || I8) { while (!mbar_try_wait(dbar, 0)) {} }                 // the epilogue warp waited
  else if (n_vp > 0) dep_wait(a, lane);
  const uint16_t* xs_row[NB8];
#pragma unroll
  for (int nb = 0; nb < NB8; ++nb) xs_row[nb] = xs + (size_t)xrow(a, gid + 8 * nb) * xs_ld + 8 * tig;

  int c_slot = 0;          // consumer ring position: slot and mbarrier phase
  uint32_t c_ph = 0;
  // release the consumed slot to the producer warp: every lane arrives after its own reads (the empty
  // barrier counts 32), so no warp-wide sync is needed
  auto advance = [&]() {
    mbar_arrive(&ebars[c_slot]);
    if (++c_slot == kNBuf) { c_slot = 0; c_ph ^= 1u; }
  };
  // ---- rank projection share: t[cc][col][rank] += V pieces · x   (64-bit fixed point, exact adds).
  // Runs before the x' staging below (it reads bf16 x from L2): t is on the critical path of every
  // epilogue.  Partials of consecutive pieces of one chunk are summed in registers before the atomics.
  {
    float tp[NB8][4];
    // fp8 factors: t_j = v_scale_j · Σ_k e4m3(V[j][k])·x_k; the scales of the current chunk's ranks gid and
    // gid + 8 are loaded when the chunk starts (off the atomics' critical path)
    float vsc[2] = {1.f, 1.f};
    auto load_vsc = [&](int cc) {
      if constexpr (F8) {
        const DMember& mv = a.m[member_of_chunk(a, cc)];
        vsc[0] = mv.vs[16 * (cc - mv.chunk_begin) + gid];
        vsc[1] = mv.vs[16 * (cc - mv.chunk_begin) + gid + 8];
      }
    };
    auto flush = [&](int cc) {
#pragma unroll
      for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = 2 * tig + (e & 1) + 8 * nb, rank = gid + 8 * (e >> 1);
          if (col < a.B) tacc_add(a.tacc, a.n_chunks, cc, col, rank, F8 ? tp[nb][e] * vsc[e >> 1] : tp[nb][e]);
          tp[nb][e] = 0.f;
        }
    };
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) tp[nb][e] = 0.f;
    int cc_cur = -1;
    for (int vp = vp0; vp < vp1; ++vp) {
      const int s = c_slot;
      const uint32_t ph = c_ph;
      int g, part;
      if constexpr (F8) v_piece8(a, vp, g, part); else v_piece(a, vp, g, part);
      const int cc = vp / ((F8 ? 2 : 4) * a.G);
      if (cc != cc_cur) {
        if (cc_cur >= 0) flush(cc_cur);
        cc_cur = cc;
        load_vsc(cc);
      }
      if constexpr (F8) {                                // 16 ranks x 64 k: two 32-k x runs per lane
        uint4 xa[NB8], xb[NB8];
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb) {
          const uint4* p = reinterpret_cast<const uint4*>(a.x + (size_t)xrow(a, gid + 8 * nb) * a.ldx + 8 * tig +
                                                          g * kGroup + 64 * part);
          xa[nb] = __ldcg(p);
          xb[nb] = __ldcg(p + 4);
        }
        while (!mbar_try_wait(&bars[s], ph)) {}
        v_tile8<NB8>(bufs + s * kBlk, lane, xa, xb, tp);
      } else {
        uint4 xv[NB8];
#pragma unroll
        for (int nb = 0; nb < NB8; ++nb) {
          const uint4* p = reinterpret_cast<const uint4*>(a.x + (size_t)xrow(a, gid + 8 * nb) * a.ldx + 8 * tig +
                                                          g * kGroup + 32 * part);
          xv[nb] = __ldcg(p);                            // bf16 x from L2 (written by the producer window)
        }
        while (!mbar_try_wait(&bars[s], ph)) {}
        v_tile<NB8>(bufs + s * kBlk, lane, xv, tp);
      }
      if (vp == vp0 && warp == 0 && lane == 0) dtrace(a, 9);     // first V piece contracted (x loaded)
      advance();
    }
    if (cc_cur >= 0) flush(cc_cur);
  }
  if (v_warp) {
    // v_done counts CTAs: the CTA's V warps meet at a named barrier, then one release add orders all
    // of their t adds before it (cumulativity through the barrier)
    asm volatile("bar.sync 7, %0;" ::"n"(kDecodeWarps * 32) : "memory");
    if (warp == 0 && lane == 0) {
      dtrace(a, 10);                                     // the CTA's V warps flushed their t atomics
      add_release(&a.cnt[0], 1u);
      dtrace(a, 12);
    }
  }
  if constexpr (I8) {
    // x (L2) -> int8 digits (smem) of this warp's groups (the same for every item: warp_share)
    if (warp == 0 && lane == 0) dtrace(a, 6);
    x8_stage(a, reinterpret_cast<uint8_t*>(xs), warp * a.G / kDecodeWarps, (warp + 1) * a.G / kDecodeWarps, lane);
    __syncwarp();
    if (warp == 0 && lane == 0) dtrace(a, 7);
  } else if constexpr (XS) {
    while (!mbar_try_wait(xbar, 0)) {}
    // in place: x (bf16) -> x' = x·2^-(fp+σ) (fp16, the B operand of the W mma); 16 elements per thread,
    // the 8 threads of one (group, batch row) are 8 consecutive lanes (they agree on σ, R20)
    const int tid = threadIdx.x;   // 0..255 (tile warps)
    for (int i = tid; i < a.G * a.B * 8; i += kDecodeWarps * 32) {
      const int part = i & 7, gb = i >> 3, b = gb % a.B, g = gb / a.B;
      uint4* src = reinterpret_cast<uint4*>(xs + (size_t)b * xs_ld + g * kGroup + part * 16);
      const uint4 in[2] = {src[0], src[1]};
      const unsigned m8 = 0xFFu << (lane & 24);
      uint32_t m = max(absmax8(in[0]), absmax8(in[1]));
      m = max(m, __shfl_xor_sync(m8, m, 1));
      m = max(m, __shfl_xor_sync(m8, m, 2));
      m = max(m, __shfl_xor_sync(m8, m, 4));
      const int sig = prescale_sigma(m);
      uint4 out[2];
      xprime16<BITS>(in, part, out, sig);
      src[0] = out[0]; src[1] = out[1];
      if (part == 0) {
        fsg[g * a.B + b] = pow2i(sig);
        if (sig != 0) misc[0] = 1u;
      }
    }
    asm volatile("bar.sync 5, %0;" ::"n"(kDecodeWarps * 32) : "memory");   // tile warps only
  }
  // fp16-path B-operand prescale (R20): factors 2^σ per (group, batch row) from the staging (XS), the
  // x-prep kernel (global), or computed per record from bf16 x (hand-off slow path); else none
  const float* fsig = nullptr;
  uint64_t slow = 0;      // x' hand-off: bit t = this warp's group g0 + t needs σ != 0 (per-record slow path)
  if constexpr (!I8) {
    if constexpr (XS) fsig = misc[0] ? fsg : nullptr;
    else if (!a.x16_given) fsig = a.xsig;
    else if (a.x16_max) {
      const int g0 = warp * a.G / kDecodeWarps, ng = (warp + 1) * a.G / kDecodeWarps - g0;
      for (int i = lane; i < ng * a.B; i += 32)
        if (prescale_sigma(__ldcg(a.x16_max + (g0 + i / a.B) * 16 + i % a.B)) != 0) slow |= 1ull << (i / a.B);
      const uint32_t lo = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)slow), hi = __reduce_or_sync(0xFFFFFFFFu, (uint32_t)(slow >> 32));
      slow = ((uint64_t)hi << 32) | lo;
    }
  }
  int k = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x, ++k) {
    const int par = k & 1;
    // this warp's groups of every item: [g0, g0 + n) (warp_share; independent of the item)
    const struct { int n, g0; } sh = {(warp + 1) * a.G / kDecodeWarps - warp * a.G / kDecodeWarps, warp * a.G / kDecodeWarps};
    float tot[NB8][4];
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
      for (int e = 0; e < 4; ++e) tot[nb][e] = 0.f;
    for (int t0 = 0; t0 < sh.n; t0 += kRPB) {
      const int s = c_slot;
      const uint32_t ph = c_ph;
      const int nt = min(kRPB, sh.n - t0);
      const uint8_t* blk = bufs + s * kBlk;
      while (!mbar_try_wait(&bars[s], ph)) {}
      if (k == 0 && t0 == 0 && warp == 0 && lane == 0 && !I8) dtrace(a, 7);
      if constexpr (I8) {
        const uint8_t* x8 = reinterpret_cast<const uint8_t*>(xs);
        const int xg = x8_stride(a.B), dd = 512 * a.B;
        float (&t1)[1][4] = *reinterpret_cast<float(*)[1][4]>(&tot[0][0]);
        if (nt == kRPB) {
#pragma unroll
          for (int t = 0; t < kRPB; ++t)
            i8_tile<BITS>(blk + t * rec_bytes(BITS), lane, x8 + (size_t)(sh.g0 + t0 + t) * xg, dd, t1);
        } else {
          for (int t = 0; t < nt; ++t)
            i8_tile<BITS>(blk + t * rec_bytes(BITS), lane, x8 + (size_t)(sh.g0 + t0 + t) * xg, dd, t1);
        }
      } else {
        // one record: x' fragments (smem, global, or the slow path's own conversion) and, with a
        // prescale, the factors 2^σ of the lane's two output columns
        auto rec = [&](auto sig_c, int t) {
          constexpr bool SIG = decltype(sig_c)::value;
          const int g = sh.g0 + t0 + t;
          uint32_t xr[NB8][16];
          float fs[NB8][2];
          const uint4* xrs[NB8];
#pragma unroll
          for (int nb = 0; nb < NB8; ++nb) xrs[nb] = reinterpret_cast<const uint4*>(xs_row[nb] + g * kGroup);
          const bool sl = (slow >> (t0 + t)) & 1ull;
          if constexpr (!XS) {
            if (SIG && sl) load_x_bf16_sig<BITS, NB8>(a, g, lane, xr, fs);
            else load_x_global<NB8>(a, g, lane, xr);
          }
          if (SIG && !sl) {
#pragma unroll
            for (int nb = 0; nb < NB8; ++nb)
#pragma unroll
              for (int h = 0; h < 2; ++h) fs[nb][h] = fsig ? fsig[g * a.B + min(2 * tig + h + 8 * nb, a.B - 1)] : 1.f;
          }
          w_tile<BITS, NB8, XS, SIG>(blk + t * rec_bytes(BITS), lane, xrs, xr, tot, fs);
        };
        const bool blk_slow = ((slow >> t0) & ((1ull << nt) - 1ull)) != 0ull;
        if (fsig == nullptr && !blk_slow) {
          if (nt == kRPB) {
            // full block: the records are independent straight-line code, so their mma chains interleave
#pragma unroll
            for (int t = 0; t < kRPB; ++t) rec(std::false_type{}, t);
          } else {
            for (int t = 0; t < nt; ++t) rec(std::false_type{}, t);
          }
        } else {
          for (int t = 0; t < nt; ++t) rec(std::true_type{}, t);
        }
      }
      advance();
    }
    if constexpr (I8) i8_finish(*reinterpret_cast<float(*)[1][4]>(&tot[0][0]), lane, a.B);
    // ---- hand the partial sums to the epilogue warp
    const int rs = k % kRedSlots;
    if (k >= kRedSlots) asm volatile("bar.sync %0, %1;" ::"r"(red_empty_id(rs)), "n"(kDecodeThreads) : "memory");   // EMPTY[rs]
    float* rb_ = red + ((size_t)(rs * kDecodeWarps + warp) * 32 + lane) * 4 * NB8;
#pragma unroll
    for (int nb = 0; nb < NB8; ++nb)
      *reinterpret_cast<float4*>(rb_ + 4 * nb) = make_float4(tot[nb][0], tot[nb][1], tot[nb][2], tot[nb][3]);
    asm volatile("bar.arrive %0, %1;" ::"r"(red_full_id(rs)), "n"(kDecodeThreads) : "memory");    // FULL[rs]
  }
}

static size_t decode_smem_bytes(bool xs, bool i8, int B, int K, int n_chunks, int fwd_chunks) {
  const int nb8 = B > 8 ? 2 : 1;
  size_t s = (size_t)kDecodeWarps * kNBuf * kTPB * kTileMax + kRedSlots * kDecodeWarps * 32 * 4 * nb8 * sizeof(float) +
             2 * kUPre * 32 * 16 + (2 * kDecodeWarps * kNBuf + 8) * sizeof(uint64_t) +
             (size_t)dec_epi_warps(i8) * (n_chunks * nb8 * 32 * 16 + 512) + (size_t)fwd_chunks * 1024;
  s += 16;                                                                 // misc
  if (i8) s += (size_t)(K / kGroup) * x8_stride(B) + kX8Pad;
  else if (xs) s += (size_t)(((K / kGroup) * B + 3) & ~3) * 4 + (size_t)B * (K + 32) * 2;   // 2^σ [G][B] + x'
  return s;
}

constexpr size_t kXsMax = 48 * 1024;
constexpr size_t kSmemOptin = 227 * 1024;   // x staged in smem when B*(K+32)*2 fits this

static bool use_xs(int B, int K) { return B <= 8 && (size_t)B * (K + 32) * 2 <= kXsMax; }
bool decode_stages_x(int B, int K) { return B <= 8 && use_xs(B, K); }

// int8 path (decode_i8.cuh): 4-bit codes, B <= 2, x8 of all groups in shared memory
constexpr size_t kX8Max = 40 * 1024;
static bool use_i8(int bits, int B, int K) {
  return options().int8_path != 0 && (bits == 4 || bits == 2) && B <= 2 && (size_t)(K / kGroup) * x8_stride(B) + kX8Pad <= kX8Max;
}
bool decode_uses_i8(int bits, int B, int K) { return use_xs(B, K) && use_i8(bits, B, K); }

// x -> x' (fp16, pre-scaled per the code layout) for the !XS decode launches.
// One thread per (group, batch row, 16-element part).
template <int BITS>
__global__ void xprep_kernel(const uint16_t* __restrict__ x, int ldx, int B, int K, uint16_t* __restrict__ x16,
                             float* __restrict__ xsig, const unsigned* dep_cnt, unsigned dep_target) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (dep_cnt) {                                          // peer mode: x is gathered from every rank
    if (threadIdx.x == 0) wait_sys(dep_cnt, dep_target);
    __syncthreads();
  }
  // one thread per (group, batch row, 16-element part): the 8 parts of a (group, row) are 8 consecutive
  // lanes and agree on the group's prescale σ (R20); 2^σ -> xsig[g][b]
  const int i = blockIdx.x * blockDim.x + threadIdx.x;   // over G * B * 8
  const int n = (K / kGroup) * B * 8;                    // a multiple of 8: 8-lane groups are all in or all out
  if (i < n) {
    const int part = i & 7, gb = i >> 3, b = gb % B, g = gb / B;
    const uint4* src = reinterpret_cast<const uint4*>(x + (size_t)b * ldx + g * kGroup + part * 16);
    const uint4 in[2] = {__ldg(src), __ldg(src + 1)};
    const unsigned m8 = 0xFFu << (threadIdx.x & 24);
    uint32_t m = max(absmax8(in[0]), absmax8(in[1]));
    m = max(m, __shfl_xor_sync(m8, m, 1));
    m = max(m, __shfl_xor_sync(m8, m, 2));
    m = max(m, __shfl_xor_sync(m8, m, 4));
    const int sig = prescale_sigma(m);
    uint4 out[2];
    xprime16<BITS>(in, part, out, sig);
    uint4* dst = reinterpret_cast<uint4*>(x16 + (size_t)b * K + g * kGroup + part * 16);
    dst[0] = out[0]; dst[1] = out[1];
    if (part == 0) xsig[g * B + b] = pow2i(sig);
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

cudaError_t launch_xprep(const uint16_t* x, int ldx, int B, int K, int bits, uint16_t* x16, float* xsig, cudaStream_t st,
                         const unsigned* dep_cnt, unsigned dep_target) {
  const int n = (K / kGroup) * B * 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((n + 255) / 256);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = options().pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  switch (bits) {
    case 2: return cudaLaunchKernelEx(&cfg, xprep_kernel<2>, x, ldx, B, K, x16, xsig, dep_cnt, dep_target);
    case 3: return cudaLaunchKernelEx(&cfg, xprep_kernel<3>, x, ldx, B, K, x16, xsig, dep_cnt, dep_target);
    case 4: return cudaLaunchKernelEx(&cfg, xprep_kernel<4>, x, ldx, B, K, x16, xsig, dep_cnt, dep_target);
    default: return cudaErrorInvalidValue;
  }
}

template <int BITS, int NB8, bool XS, bool I8, bool F8>
static cudaError_t launch_tf(const DArgs& a, int grid, cudaStream_t st) {
  const size_t smem = decode_smem_bytes(XS, I8, a.B, a.K, a.n_chunks, a.fwd ? a.fwd_chunks : 0);
  if (smem > kSmemOptin) return cudaErrorInvalidConfiguration;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<BITS, NB8, XS, I8, F8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemOptin);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(dec_block(I8));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = options().pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, decode_kernel<BITS, NB8, XS, I8, F8>, a);
}
// fp8 factors select their own instantiation (no run-time branch in the bf16 kernels)
template <int BITS, int NB8, bool XS, bool I8>
static cudaError_t launch_t(const DArgs& a, int grid, cudaStream_t st) {
  return a.fp8 ? launch_tf<BITS, NB8, XS, I8, true>(a, grid, st) : launch_tf<BITS, NB8, XS, I8, false>(a, grid, st);
}

template <int BITS, int NB8, bool XS, bool I8>
static int max_ctas_t(int B, int K, int n_chunks, int fwd_chunks) {
  const size_t smem = decode_smem_bytes(XS, I8, B, K, n_chunks, fwd_chunks);
  cudaFuncSetAttribute(decode_kernel<BITS, NB8, XS, I8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kSmemOptin);
  cudaFuncSetAttribute(decode_kernel<BITS, NB8, XS, I8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kSmemOptin);
  int per_sm = 0, per_sm8 = 0, dev = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, decode_kernel<BITS, NB8, XS, I8, false>, dec_block(I8), smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm8, decode_kernel<BITS, NB8, XS, I8, true>, dec_block(I8), smem);
  per_sm = per_sm < per_sm8 ? per_sm : per_sm8;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;
}

#define HC_DISPATCH(FN, ...)                                                       \
  do {                                                                             \
    const bool two = a_B > 8, xs = use_xs(a_B, a_K) && !a_noxs;                   \
    switch (bits) {                                                                \
      case 2: return two ? FN<2, 2, false, false>(__VA_ARGS__)                     \
                         : (xs ? (use_i8(2, a_B, a_K) ? FN<2, 1, true, true>(__VA_ARGS__)                   \
                                                      : FN<2, 1, true, false>(__VA_ARGS__))                 \
                               : FN<2, 1, false, false>(__VA_ARGS__));                                     \
      case 3: return two ? FN<3, 2, false, false>(__VA_ARGS__)                     \
                         : (xs ? FN<3, 1, true, false>(__VA_ARGS__) : FN<3, 1, false, false>(__VA_ARGS__)); \
      case 4: return two ? FN<4, 2, false, false>(__VA_ARGS__)                     \
                         : (xs ? (use_i8(4, a_B, a_K) ? FN<4, 1, true, true>(__VA_ARGS__)                   \
                                                      : FN<4, 1, true, false>(__VA_ARGS__))                 \
                               : FN<4, 1, false, false>(__VA_ARGS__));                                     \
      default: break;                                                              \
    }                                                                              \
  } while (0)

cudaError_t launch_decode(const DArgs& a, int bits, int grid, cudaStream_t st) {
  const int a_B = a.B, a_K = a.K;
  const bool a_noxs = a.x16_given != 0;
  HC_DISPATCH(launch_t, a, grid, st);
  return cudaErrorInvalidValue;
}

int decode_max_ctas(int bits, int B, int K, int n_chunks, int fwd_chunks, bool no_xs) {
  const int a_B = B, a_K = K;
  const bool a_noxs = no_xs;
  HC_DISPATCH(max_ctas_t, B, K, n_chunks, fwd_chunks);
  return 0;
}

}  // namespace hc
