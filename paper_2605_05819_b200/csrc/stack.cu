// Persistent decode-stack kernel (hc_stack_forward, B <= 8, x staged in shared memory).
//
// The per-window decode kernel (decode.cu) pays a launch, a prologue and a pipeline drain at every
// window boundary (128 windows per Llama-2-7B token).  Here one launch runs the whole plan:
//  * one CTA per SM: 16 tile warps (each its own TMA bulk-copy ring) + 1 epilogue warp;
//  * every tile warp's producer streams its tiles window after window — V pieces of window w, then
//    its share (K/16 groups) of the CTA's row blocks of w, then window w + 1 ... — depending only on
//    ring slots, never on activations, so HBM keeps streaming across window boundaries while the
//    consumers wait for the previous window's output;
//  * window w's consumers start when window w-1 is complete: a device counter done[w-1] reaches
//    n_rb(w-1) (each CTA adds its row-block count once, after its last epilogue of the window, with
//    release semantics); the CTA then bulk-copies x_w into shared memory and converts it to x' in place;
//  * rank projection t = V·x as in the decode kernel (64-bit fixed-point atomics, deterministic),
//    published per window through vdone[w]; epilogues acquire it once per window;
//  * row-block items of window w run on CTA (i + rot_w) % grid, rot_w rotating by the cumulative row
//    blocks so that CTAs short of work in one window are first in the next;
//  * every activation read (x for V·x, residuals) goes through L2 (ld.global.cg / TMA): buffers are
//    reused across layers inside one launch and L1 is not coherent.
// Deadlock freedom: all CTAs are co-resident (cooperative launch, grid = SMs); every warp processes
// windows in order and, inside a window, its V pieces before its row blocks, so window w's progress
// depends only on windows < w.  Spin waits trap after ~4 s instead of hanging the device.
#include <climits>

#include "decode_dev.cuh"
#include "stack.h"

namespace hc {

namespace {

#ifndef HC_STK_TRACE
#define HC_STK_TRACE 0
#endif
// dev tracing: globaltimer stamps per (window, CTA): [0] x ready seen, [1] x' staged, [2] tiles done,
// [3] epilogue done (written to trace_buf, a __device__ pointer set by hc_stack_trace_buffer)
__device__ unsigned long long* g_trace = nullptr;
__device__ unsigned long long* g_acct = nullptr;   // [grid][17 warps][4]: data wait, EMPTY wait, x wait, total
__device__ __forceinline__ void trace(int w, int c, int ev) {
#if HC_STK_TRACE
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (g_trace) g_trace[((size_t)w * gridDim.x + c) * 4 + ev] = t;
#endif
}

constexpr int kSBlk = kSTPB * kTileMax;
constexpr int kSUMax = 8;                // U prefetch slots (items in flight) at most
constexpr int kBarTile = 9;              // named barrier of the 16 tile warps (FULL 1..4, EMPTY 5..8)


// Poll with relaxed loads (an acquire load invalidates the SM's L1 on every iteration, which evicts
// the window table the other warps are reading) and acquire once the count is reached.
__device__ __forceinline__ void wait_geq(const unsigned* p, unsigned target) {
  if (ld_relaxed(p) < target) {
    const long long t0 = clock64();
    do {
      __nanosleep(32);
      if (clock64() - t0 > (1ll << 33)) __trap();   // ~4 s: a bug, not a wait — fail loudly
    } while (ld_relaxed(p) < target);
  }
  (void)ld_acquire(p);
}


// warp-cooperative copy of one window descriptor into shared memory (the table is read-only in the
// kernel; smem copies keep the hot per-item reads off L1/L2, whose L1 share is small next to ~200 KB
// of shared memory)
__device__ __forceinline__ void load_swin(SWin* dst, const SWin* src, int lane) {
  static_assert(sizeof(SWin) % 8 == 0, "SWin copy granularity");
  constexpr int n = (int)(sizeof(SWin) / 8);
  for (int i = lane; i < n; i += 32)
    reinterpret_cast<unsigned long long*>(dst)[i] = __ldg(reinterpret_cast<const unsigned long long*>(src) + i);
  __syncwarp();
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

__device__ __forceinline__ void vrange(const SWin& W, int gw, int& vp0, int& vp1) {
  const int n_vp = W.a.n_chunks * 4 * W.a.G;
  if (gw < W.n_vwarps) {
    vp0 = (int)((long long)gw * n_vp / W.n_vwarps);
    vp1 = (int)((long long)(gw + 1) * n_vp / W.n_vwarps);
  } else {
    vp0 = vp1 = 0;
  }
}

}  // namespace

template <int BITS>
__global__ void __launch_bounds__(kSThreads, 1) stack_kernel(const __grid_constant__ StackArgs S) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int c = blockIdx.x, grid = gridDim.x;
  float* red = reinterpret_cast<float*>(smem + (size_t)kSW * kSNBuf * kSBlk);       // [kSRed][kSW][32][4]
  uint64_t* bars_all = reinterpret_cast<uint64_t*>(red + kSRed * kSW * 32 * 4);
  uint64_t* ubar = bars_all + kSW * kSNBuf;     // [kSUMax]
  uint64_t* xbar = ubar + kSUMax;               // [1]
  SWin* wc = reinterpret_cast<SWin*>(bars_all + kSW * kSNBuf + kSUMax + 2);      // [3] window copies
  uint4* tsm = reinterpret_cast<uint4*>(reinterpret_cast<uint8_t*>(wc) + 3 * ((sizeof(SWin) + 15) & ~(size_t)15));  // [kMaxChunks][32] t hi|lo
  uint4* ubuf = tsm + kMaxChunks * 32;                                              // [n_uslots][u_slot_chunks][32]
  uint16_t* xs = reinterpret_cast<uint16_t*>(ubuf + (size_t)S.n_uslots * S.u_slot_chunks * 32);   // [B][xs_ld] x'

  if (lane == 0) {
    if (warp < kSW) {
#pragma unroll
      for (int s = 0; s < kSNBuf; ++s) mbar_init(&bars_all[warp * kSNBuf + s], 1);
    } else {
      for (int j = 0; j < kSUMax; ++j) mbar_init(&ubar[j], 1);
      mbar_init(xbar, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == kSW) {
    // ======================= epilogue warp =======================
    int n_total = 0;
    for (int w = 0; w < S.n_win; ++w) {
      const int r = cta_rank(S.wins[w], c, grid), n = S.wins[w].a.n_rb;
      if (r < n) n_total += (n - r + grid - 1) / grid;
    }
    // U fragments: a ring of n_uslots item slots, filled n_uslots - 1 items ahead of the epilogue
    const int n_us = S.n_uslots;
    int uw = 0, uitem = 0, uk = 0;                    // prefetch cursor: (window, item) of item uk
    seek(S, c, grid, uw, uitem);
    int cuw = -1;                                     // window cached in wc[1]
    auto prefetch_next = [&]() {
      if (uk >= n_total) return;
      if (cuw != uw) { load_swin(&wc[1], &S.wins[uw], lane); cuw = uw; }
      const DArgs& A = wc[1].a;
      const DMember& m = A.m[member_of_rb(A, uitem)];
      const int r_eff = A.glue ? max(A.m[0].r, A.m[1].r) : m.r;
      const int nck = (r_eff + 15) >> 4;
      if (nck > 0 && lane == 0) {
        const int j = uk % n_us;
        const uint32_t bytes = (uint32_t)nck * 512u;
        mbar_expect_tx(&ubar[j], bytes);
        bulk_copy(ubuf + (size_t)j * S.u_slot_chunks * 32, m.U + (size_t)(uitem - m.rb_begin) * (m.r_stored >> 4) * 32,
                  bytes, &ubar[j], evict_first_policy());
      }
      ++uk;
      uitem += grid;
      if (uitem >= A.n_rb) { ++uw; seek(S, c, grid, uw, uitem); }
    };
    for (int j = 0; j + 1 < n_us; ++j) prefetch_next();
    unsigned u_phase = 0;                             // bit j: parity of ubar[j]
    int w = 0, item = 0;
    seek(S, c, grid, w, item);
    int t_w = -1, cnt_w = 0, cw = -1;                 // cw: window cached in wc[0]
    long long e_full = 0, e_t = 0, e_u = 0;
    const long long e_t0 = clock64();
    for (int k = 0; k < n_total; ++k) {
      const int par = k % kSRed, uj = k % n_us;
      prefetch_next();                                // item k + n_us - 1 into the slot item k - 1 freed
      if (cw != w) { load_swin(&wc[0], &S.wins[w], lane); cw = w; }
      const SWin& W = wc[0];
      const DArgs& A = W.a;
      const DMember& m = A.m[member_of_rb(A, item)];
      const int r_eff = A.glue ? max(A.m[0].r, A.m[1].r) : m.r;
      if (r_eff > 0 && t_w != w) {
        // once per CTA and window: acquire t (every V warp of the window has added its share) and keep
        // it as the bf16 hi + lo B-fragments of the U·t mma (ranks >= the member's r masked to 0)
        const long long q1 = clock64();
        if (lane == 0) wait_geq(&S.vdone[w], (unsigned)W.n_vwarps);
        __syncwarp();
        e_t += clock64() - q1;
        for (int cc = 0; cc < A.n_chunks; ++cc) {
          const DMember& mt = A.m[member_of_chunk(A, cc)];
          const int r0 = 16 * (cc - mt.chunk_begin) + 2 * tig;
          const long long* src = A.tacc + ((size_t)cc * 16 + gid) * 16 + 2 * tig;
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
        t_w = w;
      }
      const long long q0 = clock64();
      asm volatile("bar.sync %0, %1;" ::"r"(1 + par), "n"(kSThreads) : "memory");   // FULL[par]
      e_full += clock64() - q0;
      if (lane == 0 && item + grid >= A.n_rb) trace(w, c, 2);   // FULL of this CTA's last item of w
      // residual: only now is its producer window known complete (this CTA's tile warps staged x of
      // window w, i.e. window w-1 and everything before it is done; the epilogue alone may run ahead
      // of windows in which this CTA has no row blocks)
      float res[4] = {0.f, 0.f, 0.f, 0.f};
      if (A.resid && !A.glue) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int b = min(2 * tig + (e & 1), A.B - 1);
          const int n = m.row_off + (item - m.rb_begin) * kRows + gid + 8 * (e >> 1);
          res[e] = bf16_bits_to_f32(__ldcg(A.resid + (size_t)b * A.ld_resid + n));
        }
      }
      float fin[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
      for (int tw = 0; tw < kSW; ++tw) {              // fixed order: deterministic
        const float4 v = *reinterpret_cast<const float4*>(red + ((size_t)(par * kSW + tw) * 32 + lane) * 4);
        fin[0] += v.x; fin[1] += v.y; fin[2] += v.z; fin[3] += v.w;
      }
      if (k + kSRed < n_total)
        asm volatile("bar.arrive %0, %1;" ::"r"(1 + kSRed + par), "n"(kSThreads) : "memory");   // EMPTY[par]

      // ---- row-block epilogue: + U[:, :r]·t, residual / SiLU glue, output
      const int rbl = item - m.rb_begin;
      float comp[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      if (r_eff > 0) {
        const int nck = (r_eff + 15) >> 4;
        const long long q2 = clock64();
        while (!mbar_try_wait(&ubar[uj], (u_phase >> uj) & 1u)) {}
        e_u += clock64() - q2;
        u_phase ^= 1u << uj;
        for (int cch = 0; cch < nck; ++cch) {
          const uint4 u = ubuf[((size_t)uj * S.u_slot_chunks + cch) * 32 + lane];
          const uint32_t af[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 1 && !A.glue) break;
            const DMember& mt = A.glue ? A.m[h] : m;
            if (16 * cch >= mt.r) continue;
            const uint4 q = tsm[(mt.chunk_begin + cch) * 32 + lane];
            mma16816(comp[h], af, q.x, q.y);          // U·t_hi
            mma16816(comp[h], af, q.z, q.w);          // U·t_lo
          }
        }
      }
      if (A.glue) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int b = 2 * tig + e;
          if (b >= A.B) continue;
          const float up = fin[e] + comp[0][e];
          const float gt = fin[e + 2] + comp[1][e + 2];
          const float v = up * (gt / (1.f + __expf(-gt)));
          const int n = m.row_off + rbl * 8 + gid;
          if (A.y_bf16) reinterpret_cast<uint16_t*>(A.y)[(size_t)b * A.ldy + n] = (uint16_t)f32_to_bf16_rn(v);
          else          reinterpret_cast<float*>(A.y)[(size_t)b * A.ldy + n] = v;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int b = 2 * tig + (e & 1);
          if (b >= A.B) continue;
          const int n = m.row_off + rbl * kRows + gid + 8 * (e >> 1);
          float v = fin[e] + comp[0][e];
          v += res[e];
          if (A.y_bf16) reinterpret_cast<uint16_t*>(A.y)[(size_t)b * A.ldy + n] = (uint16_t)f32_to_bf16_rn(v);
          else          reinterpret_cast<float*>(A.y)[(size_t)b * A.ldy + n] = v;
        }
      }
      ++cnt_w;
      item += grid;
      if (item >= A.n_rb) {
        // this CTA's last row block of window w: publish its count (release); the CTA completing the
        // window zeroes the t accumulators for the next launch (every reader of t is done by then)
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) {
          const unsigned old = add_release(&S.done[w], (unsigned)cnt_w);
          last = (old + (unsigned)cnt_w == (unsigned)A.n_rb);
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (lane == 0) trace(w, c, 3);
        if (last)
          for (int i = lane; i < A.n_chunks * 256; i += 32) A.tacc[i] = 0;
        cnt_w = 0;
        ++w;
        seek(S, c, grid, w, item);
      }
    }
#if HC_STK_TRACE
    if (lane == 0 && g_acct) {
      unsigned long long* o = g_acct + ((size_t)c * (kSW + 1) + kSW) * 8;
      o[0] = e_full; o[1] = e_t; o[2] = e_u; o[3] = clock64() - e_t0;
    }
#endif
    return;
  }

  // ======================= tile warps =======================
  uint8_t* bufs = smem + (size_t)warp * kSNBuf * kSBlk;
  uint64_t* bars = bars_all + warp * kSNBuf;
  const uint64_t pol_w = evict_first_policy();
  // ---- producer (lane 0 issues; state is warp-uniform): V pieces then row-block shares, window by window
  int p_w = 0, p_vp = 0, p_vp1 = 0, p_item = 0, p_t = 0;
  Share p_sh{nullptr, 0, 1024, 0, 0, 0};
  auto p_enter = [&](int w) {
    p_w = w;
    if (w >= S.n_win) return;
    const SWin& W = S.wins[w];
    const int rank = cta_rank(W, c, grid);
    vrange(W, rank * kSW + warp, p_vp, p_vp1);
    p_item = rank;
    p_t = 0;
    if (p_item < W.a.n_rb) p_sh = warp_share<BITS, kSW>(W.a, p_item, warp);
  };
  unsigned blk_issued = 0;
  auto issue_block = [&]() {
    while (p_w < S.n_win) {
      const DArgs& A = S.wins[p_w].a;
      const int s = blk_issued % kSNBuf;
      if (p_vp < p_vp1) {
        int g, part;
        const uint8_t* src = v_piece(A, p_vp, g, part);
        if (lane == 0) {
          mbar_expect_tx(&bars[s], 1024u);
          bulk_copy(bufs + s * kSBlk, src, 1024u, &bars[s], pol_w);
        }
        ++p_vp;
        ++blk_issued;
        return;
      }
      while (p_item < A.n_rb && p_t >= p_sh.n) {
        p_item += grid;
        p_t = 0;
        if (p_item < A.n_rb) p_sh = warp_share<BITS, kSW>(A, p_item, warp);
      }
      if (p_item < A.n_rb) {
        const int nt = min(kSTPB, p_sh.n - p_t);
        if (lane == 0) {
          const uint32_t bytes = (uint32_t)(nt * p_sh.tb);
          mbar_expect_tx(&bars[s], bytes);
          bulk_copy(bufs + s * kSBlk, p_sh.base + (size_t)p_t * p_sh.tb, bytes, &bars[s], pol_w);
        }
        p_t += nt;
        ++blk_issued;
        return;
      }
      p_enter(p_w + 1);
    }
  };
  p_enter(0);
#pragma unroll 1
  for (int s = 0; s < kSNBuf; ++s) issue_block();

  unsigned blk_done = 0, xphase = 0;
  int k = 0;                                           // item counter of this CTA (hand-off slot)
  long long a_data = 0, a_empty = 0, a_x = 0, a_v = 0, a_bar = 0, a_st = 0;
  const long long a_t0 = clock64();
  for (int w = 0; w < S.n_win; ++w) {
    const SWin& W = S.wins[w];
    const DArgs& A = W.a;
    const int rank = cta_rank(W, c, grid);
    int vp0, vp1;
    vrange(W, rank * kSW + warp, vp0, vp1);
    // ---- rank projection share of window w (x from L2; t in 2^-28 fixed point, exact adds)
    const long long qv = clock64();
    if (rank * kSW + warp < W.n_vwarps) {             // a V warp of window w (its share may be empty)
      if (lane == 0 && w > 0) wait_geq(&S.done[w - 1], (unsigned)S.wins[w - 1].a.n_rb);
      __syncwarp();
      for (int vp = vp0; vp < vp1; ++vp) {
        const int s = blk_done % kSNBuf;
        const uint32_t ph = (blk_done / kSNBuf) & 1u;
        int g, part;
        v_piece(A, vp, g, part);
        const int cc = vp / (4 * A.G);
        uint4 xv[1];
        xv[0] = __ldcg(reinterpret_cast<const uint4*>(A.x + (size_t)xrow(A, gid) * A.ldx + 8 * tig + g * kGroup + 32 * part));
        while (!mbar_try_wait(&bars[s], ph)) {}
        float tp[1][4] = {{0.f, 0.f, 0.f, 0.f}};
        v_tile<1>(bufs + s * kSBlk, lane, xv, tp);
        __syncwarp();
        ++blk_done;
        issue_block();
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = 2 * tig + (e & 1), rk = gid + 8 * (e >> 1);
          if (col < A.B)
            atomicAdd(reinterpret_cast<unsigned long long*>(A.tacc + ((size_t)cc * 16 + col) * 16 + rk),
                      (unsigned long long)__float2ll_rn(tp[0][e] * kTScale));
        }
      }
      __syncwarp();
      if (lane == 0) add_release(&S.vdone[w], 1u);
    }
    a_v += clock64() - qv;
    if (rank >= A.n_rb) continue;                      // no row blocks of window w on this CTA

    // ---- stage x_w' in shared memory (every tile warp is past the previous window's tiles)
    const long long qb = clock64();
    asm volatile("bar.sync %0, %1;" ::"n"(kBarTile), "n"(kSW * 32) : "memory");
    a_bar += clock64() - qb;
    const long long qs = clock64();
    if (warp == 1) load_swin(&wc[2], &S.wins[w], lane);   // published by the second barrier below
    if (warp == 0 && lane == 0) {
      if (w > 0) wait_geq(&S.done[w - 1], (unsigned)S.wins[w - 1].a.n_rb);
      asm volatile("fence.proxy.async.global;" ::: "memory");
      mbar_expect_tx(xbar, (uint32_t)(A.B * A.K * 2));
      for (int b = 0; b < A.B; ++b)
        bulk_copy(xs + (size_t)b * S.xs_ld, A.x + (size_t)b * A.ldx, (uint32_t)(A.K * 2), xbar, evict_last_policy());
    }
    if (warp == 0 && lane == 0) trace(w, c, 0);
    {
      const long long q0 = clock64();
      while (!mbar_try_wait(xbar, xphase)) {}
      a_x += clock64() - q0;
    }
    xphase ^= 1u;
    for (int i = threadIdx.x; i < A.G * A.B * 8; i += kSW * 32) {
      const int part = i & 7, gb = i >> 3, b = gb % A.B, g = gb / A.B;
      uint4* src = reinterpret_cast<uint4*>(xs + (size_t)b * S.xs_ld + g * kGroup + part * 16);
      const uint4 in[2] = {src[0], src[1]};
      uint4 out[2];
      xprime16<BITS>(in, part, out);
      src[0] = out[0]; src[1] = out[1];
    }
    asm volatile("bar.sync %0, %1;" ::"n"(kBarTile), "n"(kSW * 32) : "memory");
    a_st += clock64() - qs;
    if (warp == 0 && lane == 0) trace(w, c, 1);
    const uint16_t* xs_row = xs + (size_t)xrow(A, gid) * S.xs_ld + 8 * tig;
    const DArgs& Ac = wc[2].a;

    for (int item = rank; item < Ac.n_rb; item += grid, ++k) {
      const int par = k % kSRed;
      const Share sh = warp_share<BITS, kSW>(Ac, item, warp);
      float tot[1][4] = {{0.f, 0.f, 0.f, 0.f}};
      for (int t0 = 0; t0 < sh.n; t0 += kSTPB) {
        const int s = blk_done % kSNBuf;
        const uint32_t ph = (blk_done / kSNBuf) & 1u;
        const int nt = min(kSTPB, sh.n - t0);
        const uint8_t* blk = bufs + s * kSBlk;
        {
          const long long q0 = clock64();
          while (!mbar_try_wait(&bars[s], ph)) {}
          a_data += clock64() - q0;
        }
        const uint32_t xr_unused[1][16] = {};
        if (nt == kSTPB) {
#pragma unroll
          for (int t = 0; t < kSTPB; ++t) {
            const uint4* const xrs[1] = {reinterpret_cast<const uint4*>(xs_row + (sh.g0 + t0 + t) * kGroup)};
            w_tile<BITS, 1, true>(blk + t * rec_bytes(BITS), lane, xrs, xr_unused, tot);
          }
        } else {
          for (int t = 0; t < nt; ++t) {
            const uint4* const xrs[1] = {reinterpret_cast<const uint4*>(xs_row + (sh.g0 + t0 + t) * kGroup)};
            w_tile<BITS, 1, true>(blk + t * rec_bytes(BITS), lane, xrs, xr_unused, tot);
          }
        }
        __syncwarp();
        ++blk_done;
        issue_block();
      }
      // ---- hand the partial sums to the epilogue warp
      {
        const long long q0 = clock64();
        if (k >= kSRed) asm volatile("bar.sync %0, %1;" ::"r"(1 + kSRed + par), "n"(kSThreads) : "memory");   // EMPTY[par]
        a_empty += clock64() - q0;
      }
      *reinterpret_cast<float4*>(red + ((size_t)(par * kSW + warp) * 32 + lane) * 4) =
          make_float4(tot[0][0], tot[0][1], tot[0][2], tot[0][3]);
      asm volatile("bar.arrive %0, %1;" ::"r"(1 + par), "n"(kSThreads) : "memory");                       // FULL[par]
    }
  }
#if HC_STK_TRACE
  if (lane == 0 && g_acct) {
    unsigned long long* o = g_acct + ((size_t)c * (kSW + 1) + warp) * 8;
    o[0] = a_data; o[1] = a_empty; o[2] = a_x; o[3] = clock64() - a_t0; o[4] = a_v; o[5] = a_bar; o[6] = a_st;
  }
#endif
}

cudaError_t stack_set_trace(void* buf) { return cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf)); }
cudaError_t stack_set_acct(void* buf) { return cudaMemcpyToSymbol(g_acct, &buf, sizeof(buf)); }

size_t stack_smem_bytes(int B, int k_max, int u_slot_chunks, int n_uslots) {
  const size_t s = (size_t)kSW * kSNBuf * kSBlk + (size_t)kSRed * kSW * 32 * 4 * sizeof(float) +
                   (size_t)(kSW * kSNBuf + kSUMax + 2) * sizeof(uint64_t) + 3 * ((sizeof(SWin) + 15) & ~(size_t)15) +
                   (size_t)kMaxChunks * 32 * 16 +
                   (size_t)n_uslots * u_slot_chunks * 512 + (size_t)B * (k_max + 32) * 2;
  return s <= 227 * 1024 ? s : 0;
}

int stack_uslots_max() { return kSUMax; }

int stack_vwarps(int n_vp, int grid) {
  if (n_vp <= 0) return 0;
  const int ctas = (n_vp + kSW * kVPerWarp - 1) / (kSW * kVPerWarp);
  return (ctas < grid ? ctas : grid) * kSW;
}

template <int BITS>
static int grid_t(size_t smem) {
  if (cudaFuncSetAttribute(stack_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return 0;
  int per_sm = 0, dev = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, stack_kernel<BITS>, kSThreads, smem) != cudaSuccess) return 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return per_sm >= 1 ? sms : 0;                     // one CTA per SM (deadlock freedom needs co-residency)
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
  cfg.blockDim = dim3(kSThreads);
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
