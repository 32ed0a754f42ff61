// Persistent decode-stack kernel (hc_stack_forward with HC_STACK_KERNEL=1, B <= 8).
//
// The per-window decode graph (decode.cu) is limited at window boundaries by CTA residency: the next
// window's CTAs only become resident (and start streaming their weights) when the current window's CTAs
// exit.  Here the SAME CTA structure as the decode kernel (8 tile warps + 1 epilogue warp, 2 CTAs per
// SM) runs every window of the stack in one cooperative launch:
//  * each tile warp's producer streams its tiles window after window into its TMA bulk-copy ring,
//    depending only on ring slots — the next window's weights are in flight while the current window
//    finishes;
//  * window w's row blocks start when window w-1 is complete: the epilogue warp polls done[w-1]
//    (relaxed loads, one acquire) and releases the CTA's tile warps with a named barrier;
//  * x' (fp16, pre-scaled) is written by the producer window's epilogue (x' hand-off) and read by the
//    tile loop from L2 / L1; window 0's x' comes from the x-prep kernel launched before;
//  * t = V·x of window w + 1 is forwarded by window w's epilogues (fixed-point atomics, deterministic);
//    window 0's t comes from in-kernel rank-projection pieces (published through vdone);
//  * U·t and the residual are formed before the partial sums arrive; each CTA publishes its row-block
//    count per window with release semantics; the CTA completing a window zeroes its t accumulators.
// Deadlock freedom: all CTAs are co-resident (cooperative launch); every warp processes windows in order
// and window w's progress depends only on windows < w.  Spin waits trap after ~4 s.
#include <climits>

#include "decode_dev.cuh"
#include "stack.h"

namespace hc {

namespace {

constexpr int kSBlk = kTPB * kTileMax;

__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned target) {
  if (ld_relaxed(p) < target) {
    const long long t0 = clock64();
    do {
      __nanosleep(48);
      if (clock64() - t0 > (1ll << 33)) __trap();   // ~4 s: a bug, not a wait — fail loudly
    } while (ld_relaxed(p) < target);
  }
  (void)ld_acquire(p);
}

// x' fragments of one group from the lane's row pointer (coherent weak loads: x' is written by the
// previous window of this launch; ordered by the epilogue's acquire + bar.sync 6)
__device__ __forceinline__ void load_xp(const uint4* p, uint32_t (&xr)[1][16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 v;
    asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + 4 * q));
    xr[0][4 * q + 0] = v.x; xr[0][4 * q + 1] = v.y; xr[0][4 * q + 2] = v.z; xr[0][4 * q + 3] = v.w;
  }
}

__device__ __forceinline__ int cta_rank(const SWin& W, int c, int grid) {
  int r = (c - W.rot) % grid;
  return r < 0 ? r + grid : r;
}

// first (window, item) of CTA c at or after window w
__device__ __forceinline__ void seek(const StackArgs& S, int c, int grid, int& w, int& item) {
  for (; w < S.n_win; ++w) {
    item = cta_rank(S.wins[w], c, grid);
    if (item < S.wins[w].a.n_rb) return;
  }
  item = 0;
}

}  // namespace

template <int BITS>
__global__ void __launch_bounds__(kDecodeThreads, 2) stack_kernel(const __grid_constant__ StackArgs S) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int c = blockIdx.x, grid = gridDim.x;
  constexpr int kEpi = kDecodeWarps;
  float* red = reinterpret_cast<float*>(smem + (size_t)kDecodeWarps * kNBuf * kSBlk);  // [2][8][32][4]
  uint4* ubuf = reinterpret_cast<uint4*>(red + 2 * kDecodeWarps * 32 * 4);             // [2][kUPre][32]
  uint64_t* bars_all = reinterpret_cast<uint64_t*>(ubuf + 2 * kUPre * 32);
  uint64_t* ubar = bars_all + kDecodeWarps * kNBuf;   // [2]
  uint64_t* fbar = ubar + 2;                          // [1]
  uint4* tsm = reinterpret_cast<uint4*>(bars_all + kDecodeWarps * kNBuf + 4);          // [kMaxChunks][32]
  uint16_t* xt = reinterpret_cast<uint16_t*>(tsm + kMaxChunks * 32);                   // [16 k][16 cols]
  uint4* fbuf = reinterpret_cast<uint4*>(xt + 256);                                    // [kFwdMax][32]
  DArgs* sA = reinterpret_cast<DArgs*>(fbuf + kFwdMax * 32);                           // epilogue's window args

  if (lane == 0) {
    if (warp < kDecodeWarps) {
#pragma unroll
      for (int s = 0; s < kNBuf; ++s) mbar_init(&bars_all[warp * kNBuf + s], 1);
    } else {
      mbar_init(&ubar[0], 1); mbar_init(&ubar[1], 1); mbar_init(fbar, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  const SWin& W0 = S.wins[0];
  const int n_vp0 = W0.a.t_in ? 0 : W0.a.n_chunks * 4 * W0.a.G;

  if (warp == kEpi) {
    // ======================= epilogue warp =======================
    auto prefetch_u = [&](int w, int item, int par) {   // U fragments of (window w, item) -> ubuf[par]
      if (w >= S.n_win) return;
      const DArgs& A = S.wins[w].a;
      const DMember& m = A.m[member_of_rb(A, item)];
      const int r_eff = A.glue ? max(A.m[0].r, A.m[1].r) : m.r;
      const int nck = min((r_eff + 15) >> 4, kUPre);
      if (nck == 0) return;
      if (lane == 0) {
        const uint32_t bytes = (uint32_t)nck * 512u;
        mbar_expect_tx(&ubar[par], bytes);
        bulk_copy(ubuf + par * kUPre * 32, m.U + (size_t)(item - m.rb_begin) * (m.r_stored >> 4) * 32, bytes,
                  &ubar[par], evict_first_policy());
      }
    };
    int uw = 0, uitem = 0;
    seek(S, c, grid, uw, uitem);
    prefetch_u(uw, uitem, 0);
    unsigned u_phase = 0, f_phase = 0;
    int k = 0;
    for (int w = 0; w < S.n_win; ++w) {
      const SWin& W = S.wins[w];
      const int rank = cta_rank(W, c, grid);
      if (rank >= W.a.n_rb) continue;
      // the window's arguments in shared memory (the table is in global memory; the per-item reads
      // below would otherwise be dependent L1/L2 loads)
      for (int i = lane; i < (int)(sizeof(DArgs) / 4); i += 32)
        reinterpret_cast<uint32_t*>(sA)[i] = __ldg(reinterpret_cast<const uint32_t*>(&W.a) + i);
      __syncwarp();
      const DArgs& a = *sA;
      // window w's x' and t are ready once window w-1 is complete (t forwarded before its release)
      if (w > 0) {
        if (lane == 0) wait_geq(&S.done[w - 1], (unsigned)S.wins[w - 1].a.n_rb);
        __syncwarp();
      }
      asm volatile("bar.sync 6, %0;" ::"n"(kDecodeThreads) : "memory");   // release this CTA's tile warps
      bool t_ready = false;
      int cnt_w = 0;
      for (int item = rank; item < a.n_rb; item += grid, ++k) {
        const int par = k & 1;
        const DMember& m = a.m[member_of_rb(a, item)];
        const int r_eff = a.glue ? max(a.m[0].r, a.m[1].r) : m.r;
        if (!t_ready && r_eff > 0) {
          if (w == 0 && lane == 0) wait_geq(S.vdone, (unsigned)S.n_vwarps0);
          __syncwarp();
#pragma unroll 4
          for (int cc = 0; cc < a.n_chunks; ++cc) {
            const DMember& mt = a.m[member_of_chunk(a, cc)];
            const int r0 = 16 * (cc - mt.chunk_begin) + 2 * tig;
            const long long* src = a.tacc + ((size_t)cc * 16 + gid) * 16 + 2 * tig;
            const long long tr[4] = {__ldcg(src), __ldcg(src + 1), __ldcg(src + 8), __ldcg(src + 9)};
            uint32_t hi[2], lo[2];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float ta = (r0 + 8 * hh < mt.r) ? (float)tr[2 * hh] * kTInv : 0.f;
              const float tb = (r0 + 8 * hh + 1 < mt.r) ? (float)tr[2 * hh + 1] * kTInv : 0.f;
              const uint32_t ha = f32_to_bf16_rn(ta), hb = f32_to_bf16_rn(tb);
              hi[hh] = ha | (hb << 16);
              lo[hh] = f32_to_bf16_rn(ta - bf16_bits_to_f32(ha)) | (f32_to_bf16_rn(tb - bf16_bits_to_f32(hb)) << 16);
            }
            tsm[cc * 32 + lane] = make_uint4(hi[0], hi[1], lo[0], lo[1]);
          }
          __syncwarp();
          t_ready = true;
        }
        // t forwarding: prefetch the next window's natural-k V fragments of this item's 16-k block
        const int f_n0 = a.glue ? m.row_off + (item - m.rb_begin) * 8 : m.row_off + (item - m.rb_begin) * kRows;
        const bool f_on = a.fwd && f_n0 >= a.fwd_lo && f_n0 < a.fwd_hi;
        if (f_on && lane == 0) {
          const int kb = (f_n0 - a.fwd_lo) >> 4;
          mbar_expect_tx(fbar, (uint32_t)a.fwd_chunks * 512u);
          for (int i = 0; i < a.fwd_nm; ++i) {
            const int nc = a.fwd_cb[i + 1] - a.fwd_cb[i];
            if (nc > 0)
              bulk_copy(fbuf + a.fwd_cb[i] * 32, a.fwd_vn[i] + (size_t)kb * a.fwd_rs[i] * 32, (uint32_t)nc * 512u, fbar,
                        evict_first_policy());
          }
        }
        // ---- before the partial sums: U[:, :r]·t and the residual
        const int rbl = item - m.rb_begin;
        float comp[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        if (r_eff > 0) {
          const int nck = (r_eff + 15) >> 4;
          while (!mbar_try_wait(&ubar[par], (u_phase >> par) & 1u)) {}
          u_phase ^= 1u << par;
          for (int cch = 0; cch < nck; ++cch) {
            const uint4 u = (cch < kUPre) ? ubuf[(par * kUPre + cch) * 32 + lane]
                                          : __ldg(m.U + ((size_t)rbl * (m.r_stored >> 4) + cch) * 32 + lane);
            const uint32_t af[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h == 1 && !a.glue) break;
              const DMember& mt = a.glue ? a.m[h] : m;
              if (16 * cch >= mt.r) continue;
              const uint4 q = tsm[(mt.chunk_begin + cch) * 32 + lane];
              mma16816(comp[h], af, q.x, q.y);
              mma16816(comp[h], af, q.z, q.w);
            }
          }
        }
        float res[4] = {0.f, 0.f, 0.f, 0.f};
        if (a.resid && !a.glue) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int b = 2 * tig + (e & 1);
            if (b < a.B)
              res[e] = bf16_bits_to_f32(__ldcg(a.resid + (size_t)b * a.ld_resid + m.row_off + rbl * kRows + gid + 8 * (e >> 1)));
          }
        }
        if (f_on) {
          reinterpret_cast<uint4*>(xt)[lane] = make_uint4(0u, 0u, 0u, 0u);
          __syncwarp();
        }
        asm volatile("bar.sync %0, %1;" ::"r"(1 + par), "n"(kDecodeThreads) : "memory");   // FULL[par]
        float fin[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int tw = 0; tw < kDecodeWarps; ++tw) {        // fixed order: deterministic
          const float4 v = *reinterpret_cast<const float4*>(red + ((size_t)(par * kDecodeWarps + tw) * 32 + lane) * 4);
          fin[0] += v.x; fin[1] += v.y; fin[2] += v.z; fin[3] += v.w;
        }
        asm volatile("bar.arrive %0, %1;" ::"r"(3 + par), "n"(kDecodeThreads) : "memory");   // EMPTY[par]
        // next item's U fragments (possibly in a later window)
        uitem += grid;
        if (uw < S.n_win && uitem >= S.wins[uw].a.n_rb) { ++uw; seek(S, c, grid, uw, uitem); }
        prefetch_u(uw, uitem, par ^ 1);
        // ---- output (+ glue / residual), the next window's x', t forwarding
        if (a.glue) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int b = 2 * tig + e;
            if (b >= a.B) continue;
            const float up = fin[e] + comp[0][e];
            const float gt = fin[e + 2] + comp[1][e + 2];
            const float v = up * (gt / (1.f + __expf(-gt)));
            const int n = m.row_off + rbl * 8 + gid;
            const uint16_t bits = (uint16_t)f32_to_bf16_rn(v);
            reinterpret_cast<uint16_t*>(a.y)[(size_t)b * a.ldy + n] = bits;
            if (f_on) xt[(((f_n0 - a.fwd_lo) & 15) + gid) * 16 + b] = bits;
            if (a.y16 && n >= a.y16_lo && n < a.y16_hi) write_xprime<BITS>(a, b, n, bits);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int b = 2 * tig + (e & 1);
            if (b >= a.B) continue;
            const int n = m.row_off + rbl * kRows + gid + 8 * (e >> 1);
            const float v = fin[e] + comp[0][e] + res[e];
            const uint16_t bits = (uint16_t)f32_to_bf16_rn(v);
            reinterpret_cast<uint16_t*>(a.y)[(size_t)b * a.ldy + n] = bits;
            if (f_on) xt[(gid + 8 * (e >> 1)) * 16 + b] = bits;
            if (a.y16 && n >= a.y16_lo && n < a.y16_hi) write_xprime<BITS>(a, b, n, bits);
          }
        }
        if (f_on) {
          __syncwarp();
          const uint32_t b0 = (uint32_t)xt[(2 * tig) * 16 + gid] | ((uint32_t)xt[(2 * tig + 1) * 16 + gid] << 16);
          const uint32_t b1 = (uint32_t)xt[(2 * tig + 8) * 16 + gid] | ((uint32_t)xt[(2 * tig + 9) * 16 + gid] << 16);
          while (!mbar_try_wait(fbar, f_phase)) {}
          f_phase ^= 1u;
#pragma unroll 4
          for (int cc = 0; cc < a.fwd_chunks; ++cc) {
            const uint4 v4 = fbuf[cc * 32 + lane];
            const uint32_t af[4] = {v4.x, v4.y, v4.z, v4.w};
            float tp[4] = {0.f, 0.f, 0.f, 0.f};
            mma16816(tp, af, b0, b1);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int col = 2 * tig + (e & 1), rk = gid + 8 * (e >> 1);
              if (col < a.B)
                atomicAdd(reinterpret_cast<unsigned long long*>(a.fwd_tacc + ((size_t)cc * 16 + col) * 16 + rk),
                          (unsigned long long)__float2ll_rn(tp[e] * kTScale));
            }
          }
          __syncwarp();                                    // fbuf / xt reused by the next item
        }
        ++cnt_w;
      }
      // this CTA's row blocks of window w are complete (outputs, x', t forwarded): publish (release);
      // the CTA completing the window zeroes its t accumulators (all of its readers are done)
      __syncwarp();
      unsigned last = 0;
      if (lane == 0) {
        const unsigned old = add_release(&S.done[w], (unsigned)cnt_w);
        last = (old + (unsigned)cnt_w == (unsigned)a.n_rb);
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last)
        for (int i = lane; i < a.n_chunks * 256; i += 32) a.tacc[i] = 0;
    }
    return;
  }

  // ======================= tile warps =======================
  uint8_t* bufs = smem + (size_t)warp * kNBuf * kSBlk;
  uint64_t* bars = bars_all + warp * kNBuf;
  const uint64_t pol_w = evict_first_policy();
  // window 0 V pieces of this warp (global warp index by rank in window 0)
  const int rank0 = cta_rank(W0, c, grid);
  const int gw0 = rank0 * kDecodeWarps + warp;
  const bool v_warp = gw0 < S.n_vwarps0;
  const int vp0 = v_warp ? (int)((long long)gw0 * n_vp0 / S.n_vwarps0) : 0;
  const int vp1 = v_warp ? (int)((long long)(gw0 + 1) * n_vp0 / S.n_vwarps0) : 0;
  // ---- producer (lane 0 issues; state warp-uniform): window 0's V pieces, then row-block shares window
  // after window, limited only by ring slots
  int vp_issue = vp0;
  int p_w = 0, p_item = 0, p_t = 0;
  seek(S, c, grid, p_w, p_item);
  Share p_sh{nullptr, 0, 1024, 0, 0, 0};
  int p_nrb = 0;
  if (p_w < S.n_win) { p_sh = warp_share<BITS>(S.wins[p_w].a, p_item, warp); p_nrb = S.wins[p_w].a.n_rb; }
  unsigned blk_issued = 0;
  auto issue_block = [&]() {
    const int s = blk_issued % kNBuf;
    if (vp_issue < vp1) {
      int g, part;
      const uint8_t* src = v_piece(W0.a, vp_issue, g, part);
      if (lane == 0) {
        mbar_expect_tx(&bars[s], 1024u);
        bulk_copy(bufs + s * kSBlk, src, 1024u, &bars[s], pol_w);
      }
      ++vp_issue;
      ++blk_issued;
      return;
    }
    while (p_w < S.n_win) {
      if (p_t < p_sh.n) break;                           // fast path: the current share continues
      p_item += grid;
      p_t = 0;
      if (p_item < p_nrb) { p_sh = warp_share<BITS>(S.wins[p_w].a, p_item, warp); continue; }
      ++p_w;
      seek(S, c, grid, p_w, p_item);
      if (p_w < S.n_win) { p_sh = warp_share<BITS>(S.wins[p_w].a, p_item, warp); p_nrb = S.wins[p_w].a.n_rb; }
    }
    if (p_w >= S.n_win) return;
    const int nt = min(kTPB, p_sh.n - p_t);
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(nt * p_sh.tb);
      mbar_expect_tx(&bars[s], bytes);
      bulk_copy(bufs + s * kSBlk, p_sh.base + (size_t)p_t * p_sh.tb, bytes, &bars[s], pol_w);
    }
    p_t += nt;
    ++blk_issued;
  };
#pragma unroll 1
  for (int s = 0; s < kNBuf; ++s) issue_block();

  unsigned blk_done = 0;
  // ---- window 0 rank projection share (x from L2; t in 2^-28 fixed point, exact adds); partials of
  // consecutive pieces of one chunk summed in registers first (same grouping as decode.cu)
  {
    float tp[1][4] = {{0.f, 0.f, 0.f, 0.f}};
    auto flush = [&](int cc) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = 2 * tig + (e & 1), rk = gid + 8 * (e >> 1);
        if (col < W0.a.B)
          atomicAdd(reinterpret_cast<unsigned long long*>(W0.a.tacc + ((size_t)cc * 16 + col) * 16 + rk),
                    (unsigned long long)__float2ll_rn(tp[0][e] * kTScale));
        tp[0][e] = 0.f;
      }
    };
    int cc_cur = -1;
    for (int vp = vp0; vp < vp1; ++vp) {
      const int s = blk_done % kNBuf;
      const uint32_t ph = (blk_done / kNBuf) & 1u;
      int g, part;
      v_piece(W0.a, vp, g, part);
      const int cc = vp / (4 * W0.a.G);
      if (cc != cc_cur) {
        if (cc_cur >= 0) flush(cc_cur);
        cc_cur = cc;
      }
      uint4 xv[1];
      xv[0] = __ldcg(reinterpret_cast<const uint4*>(W0.a.x + (size_t)xrow(W0.a, gid) * W0.a.ldx + 8 * tig + g * kGroup +
                                                    32 * part));
      while (!mbar_try_wait(&bars[s], ph)) {}
      v_tile<1>(bufs + s * kSBlk, lane, xv, tp);
      __syncwarp();
      ++blk_done;
      issue_block();
    }
    if (cc_cur >= 0) flush(cc_cur);
  }
  if (v_warp) {
    __syncwarp();
    if (lane == 0) add_release(S.vdone, 1u);
  }

  int k = 0;
  for (int w = 0; w < S.n_win; ++w) {
    const DArgs& a = S.wins[w].a;
    const int rank = cta_rank(S.wins[w], c, grid);
    if (rank >= a.n_rb) continue;
    const int n_rb = a.n_rb;
    // this lane's x' row (fp16, pre-scaled) of the window: x'[xrow(gid)][8·tig ..]
    const uint4* xp = reinterpret_cast<const uint4*>(a.x16 + (size_t)xrow(a, gid) * a.K + 8 * tig);
    asm volatile("bar.sync 6, %0;" ::"n"(kDecodeThreads) : "memory");   // the epilogue warp saw window w-1 done
    for (int item = rank; item < n_rb; item += grid, ++k) {
      const int par = k & 1;
      const Share sh = warp_share<BITS>(a, item, warp);
      float tot[1][4] = {{0.f, 0.f, 0.f, 0.f}};
      for (int t0 = 0; t0 < sh.n; t0 += kTPB) {
        const int s = blk_done % kNBuf;
        const uint32_t ph = (blk_done / kNBuf) & 1u;
        const int nt = min(kTPB, sh.n - t0);
        const uint8_t* blk = bufs + s * kSBlk;
        while (!mbar_try_wait(&bars[s], ph)) {}
        const uint4* const unused[1] = {nullptr};
        if (nt == kTPB) {
#pragma unroll
          for (int t = 0; t < kTPB; ++t) {
            uint32_t xr[1][16];
            load_xp(xp + (size_t)(sh.g0 + t0 + t) * (kGroup / 8), xr);
            w_tile<BITS, 1, false>(blk + t * rec_bytes(BITS), lane, unused, xr, tot);
          }
        } else {
          for (int t = 0; t < nt; ++t) {
            uint32_t xr[1][16];
            load_xp(xp + (size_t)(sh.g0 + t0 + t) * (kGroup / 8), xr);
            w_tile<BITS, 1, false>(blk + t * rec_bytes(BITS), lane, unused, xr, tot);
          }
        }
        __syncwarp();
        ++blk_done;
        issue_block();
      }
      if (k >= 2) asm volatile("bar.sync %0, %1;" ::"r"(3 + par), "n"(kDecodeThreads) : "memory");   // EMPTY[par]
      *reinterpret_cast<float4*>(red + ((size_t)(par * kDecodeWarps + warp) * 32 + lane) * 4) =
          make_float4(tot[0][0], tot[0][1], tot[0][2], tot[0][3]);
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + par), "n"(kDecodeThreads) : "memory");            // FULL[par]
    }
  }
}

size_t stack_smem_bytes() {
  return (size_t)kDecodeWarps * kNBuf * kSBlk + 2 * kDecodeWarps * 32 * 4 * sizeof(float) + 2 * kUPre * 32 * 16 +
         (size_t)(kDecodeWarps * kNBuf + 4) * sizeof(uint64_t) + (size_t)kMaxChunks * 32 * 16 + 512 +
         (size_t)kFwdMax * 512 + (sizeof(DArgs) + 15) / 16 * 16;
}

int stack_vwarps(int n_vp, int grid) {
  if (n_vp <= 0) return 0;
  const int ctas = (n_vp + kDecodeWarps * kVPerWarp - 1) / (kDecodeWarps * kVPerWarp);
  return (ctas < grid ? ctas : grid) * kDecodeWarps;
}

template <int BITS>
static int grid_t(size_t smem) {
  if (cudaFuncSetAttribute(stack_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stack_kernel<BITS>, kDecodeThreads, smem) != cudaSuccess) return 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm * sms;                          // every CTA co-resident (the spin waits need it)
}

int stack_grid(int bits, size_t smem) {
  switch (bits) {
    case 2: return grid_t<2>(smem);
    case 3: return grid_t<3>(smem);
    case 4: return grid_t<4>(smem);
    default: return 0;
  }
}

template <int BITS>
static cudaError_t launch_t(const StackArgs& s, int grid, size_t smem, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(stack_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kDecodeThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;       // all CTAs co-resident, or the launch fails
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, stack_kernel<BITS>, s);
}

cudaError_t launch_stack(const StackArgs& s, int bits, int grid, size_t smem, cudaStream_t st) {
  switch (bits) {
    case 2: return launch_t<2>(s, grid, smem, st);
    case 3: return launch_t<3>(s, grid, smem, st);
    case 4: return launch_t<4>(s, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hc
