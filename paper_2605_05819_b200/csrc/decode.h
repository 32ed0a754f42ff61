// Fused decode kernel interface (one compensation window per launch).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hc {

constexpr int kMaxMembers = 4;
constexpr int kDecodeWarps = 8;          // tile (streaming + contraction) warps per CTA
#ifndef HC_DEC_EPI
#define HC_DEC_EPI 3
#endif
// epilogue warps per CTA: item k of a CTA goes to epilogue warp k % epi (its own reduction buffer, U buffer, named
// barriers FULL / EMPTY[k % 2] and t fragments), so the per-item epilogue work (reduction of the 8 partial sums,
// U·t, output, t forwarding) of consecutive items runs in parallel.  HC_DEC_EPI = 1 or 2 everywhere; 3 (default):
// two on the int8 path, one on the fp16 path (whose tile loop needs > 88 registers: a 12th warp would cap it there)
constexpr int dec_epi_warps(bool i8) { return HC_DEC_EPI == 3 ? (i8 ? 2 : 1) : HC_DEC_EPI; }
static_assert(HC_DEC_EPI >= 1 && HC_DEC_EPI <= 3, "HC_DEC_EPI: 1, 2 or 3");
constexpr int kDecodeThreads = (kDecodeWarps + 1) * 32;   // tile warps + one epilogue warp (named-barrier count)
#ifndef HC_DEC_RED
#define HC_DEC_RED 2   // (4 measured neutral on C2 and it costs the 2-bit C5 windows their second CTA per SM)
#endif
// reduction slots: the tile warps run up to kRedSlots items ahead of the epilogue warps (item k -> slot k % kRedSlots),
// so a window's weight stream continues while its first epilogues wait for t = V·x
constexpr int kRedSlots = HC_DEC_RED;
static_assert(kRedSlots == 2 || kRedSlots == 4, "2 or 4 reduction slots");
// named barrier ids of slot s: FULL (tile warps arrive, the epilogue warp syncs), EMPTY (the reverse)
__host__ __device__ constexpr int red_full_id(int s) { return s < 2 ? 1 + s : 6 + s; }    // 1, 2, 8, 9
__host__ __device__ constexpr int red_empty_id(int s) { return s < 2 ? 3 + s : 8 + s; }   // 3, 4, 10, 11
constexpr int dec_block(bool i8) { return (kDecodeWarps + dec_epi_warps(i8) + 1) * 32; }   // + the producer warp
constexpr int kMaxChunks = 32;           // Σ ceil(r_m/16) over a window's members
#ifndef HC_DEC_TPB
#define HC_DEC_TPB 2
#endif
#ifndef HC_DEC_NBUF
#define HC_DEC_NBUF 3
#endif
#ifndef HC_DEC_MINB
#define HC_DEC_MINB 2
#endif
constexpr int kTPB = HC_DEC_TPB;         // tiles per bulk-copy block
constexpr int kNBuf = HC_DEC_NBUF;       // block buffers per warp (kNBuf - 1 blocks in flight while one computes)
constexpr int kTileMax = 1088;           // >= rec_bytes(4) = 1072, >= 1 KB V piece
#ifndef HC_DEC_UPRE
#define HC_DEC_UPRE 8
#endif
constexpr int kUPre = HC_DEC_UPRE;       // U chunks (16 ranks each) staged in smem per item (r <= 128)
constexpr int kTTiers = 4;               // t accumulator tiers (decode_dev.cuh tacc_add)
constexpr int kTChunk = kTTiers * 256;   // t accumulator words per rank chunk: [tier][16 cols][16 ranks]
#ifndef HC_TCOPIES
#define HC_TCOPIES 1   // measured: 4 copies C1 891 vs 1189 GB/s, 8 copies 585 (the epilogue's extra loads cost more than the queue)
#endif
// t accumulator copies: a CTA adds into copy blockIdx % kTCopies and readers sum the copies, which divides the
// same-address atomic queue at L2 (every item of a window adds into the same t elements)
constexpr int kTCopies = HC_TCOPIES;
constexpr int kFwdMax = 24;              // next-window rank chunks a launch can forward t to (smem: 512 B each)

struct DMember {
  const uint8_t* rec;   // [n_rb][G][rec_bytes]          (layout.h)
  const uint4* U;       // [n_rb][r_stored/16][32]       (bf16 A-fragments of U)
  const uint4* V;       // [r_stored/16][G][8][32]       (bf16 A-fragments of V)
  int n_rb;             // local rows / 16
  int rb_begin;         // first window-global rb index
  int row_off;          // output column offset of this member inside y rows
  int r;                // allocated rank (0 = no compensation, no U/V reads)
  int r_stored;
  int chunk_begin;      // first window-global rank chunk (16 ranks) of this member
  int full_off;         // peer mode: output column (in the full, gathered window output) of local row 0
  const float* us;      // fp8 factors (DArgs::fp8): per-rank scales of U and V [r_stored]
  const float* vs;
};

constexpr int kMaxPeers = 8;

struct DArgs {
  DMember m[kMaxMembers];
  int n_members;
  int K, G, B;
  const uint16_t* x;    // bf16 [B][ldx]
  int ldx;              // row stride of x in elements (multiple of 8)
  void* y;              // [B][ldy] fp32 or bf16
  int ldy, y_bf16;
  const uint16_t* resid;  // optional bf16 [B][ld_resid] added before the output rounding
  int ld_resid;
  int glue;             // 0 none; 1 fused SiLU(gate)*up: m[0] = up (holds the interleaved records and U),
                        //   m[1] = gate (V / rank only); row block = 8 up rows + 8 gate rows
  int fp8;              // 1: U / V are e4m3 fragments (U: [rb][c][lane][8 B], V: 1 KB pieces of 16 ranks x 64 k)
                        //    with per-rank scales DMember::us / vs
  int n_rb;             // Σ members
  int n_chunks;         // Σ ceil(r_m / 16)
  const uint16_t* x16;  // !XS launches: fp16 x' = x·2^-fp [B][K] written by launch_xprep (else unused)
  int t_in;             // 1: t = V·x of this window was already accumulated into tacc by the kernel that
                        //    produced x (t forwarding); the launch runs no rank-projection pieces
  // t forwarding to the next window (the one whose input x' is this window's output):
  //   t_next[c][col][rank] += Σ_k Vn[c][k/16] · y[col][k]   for output columns k in [fwd_lo, fwd_hi)
  int fwd;              // 0 off, 1 on
  int fwd_lo, fwd_hi;   // output columns of this window that are the next window's x (k = col - fwd_lo)
  int fwd_chunks;       // Σ ceil(r/16) over the next window's members
  const uint4* fwd_vn[kMaxMembers];   // natural-k V fragments [K/16][r_stored/16][32] of the next members
  int fwd_cb[kMaxMembers + 1];        // chunk ranges: member i owns next-window chunks [fwd_cb[i], fwd_cb[i+1])
  int fwd_rs[kMaxMembers];            // r_stored / 16 of the next members (chunk stride of fwd_vn)
  int fwd_nm;           // next window's member count
  long long* fwd_tacc;  // next window's t accumulators
  int trace_slot;       // dev (HC_DEC_TRACE builds): row of the timestamp trace this launch writes
  // dataflow dependency on the producer window (stack graphs): instead of griddepcontrol.wait (the
  // kernel-boundary release, ~2 µs), wait until the producer's row-block counter reaches its n_rb
  // (release / acquire), and reset that counter when this window completes
  unsigned* dep_cnt;    // producer's cnt[1] (peer mode: this rank's gather counter), or NULL (griddepcontrol.wait)
  unsigned dep_target;  // producer's n_rb
  int keep_done;        // 1: a consumer window resets this window's cnt[1] (do not self-reset it)
  // x' hand-off (stack graphs): x16_given = 1 means x16 was written by the producer window's epilogue
  // (no x-prep kernel, no shared-memory staging: the tile warps read x' fragments from L2 / L1);
  // y16 (if set) receives this window's output columns [y16_lo, y16_hi) as the next window's x' =
  // fp16(y·2^-fp), row stride y16_hi - y16_lo
  int x16_given;
  uint16_t* y16;
  int y16_lo, y16_hi;
  // x' range (R20): the producer publishes, per (group of 128 x' columns, batch row), the largest
  // |x| (bf16 bits without sign) of its hand-off through atomicMax into y16_max [G][16]; the consumer reads
  // x16_max after its dependency wait and, for the groups whose prescale σ is not 0, builds x' itself from
  // bf16 x (per-record slow path).  clr_max[0 .. clr_n) is zeroed by CTA 0 after its dependency wait: the
  // max buffer the NEXT window publishes into (its previous reader finished before this window's producer)
  // peer mode (column sharding over G GPUs with the gather fused into the epilogue):
  // every output element is stored into each of the npeer ranks' full-width window output ypeer[q] (peer memory over
  // NVLink), the next window's t partials of this rank's output slice are added into each rank's t
  // accumulators fwdpeer[q], and each CTA adds its row-block count to each rank's dependency counter
  // dpeer[q] (system-scope release); the consumer waits for npeer x n_rb.  npeer <= 1: off.
  int npeer;
  uint16_t* ypeer[kMaxPeers];
  int ld_full;          // row stride of ypeer (the full window output width)
  unsigned* dpeer[kMaxPeers];
  long long* fwdpeer[kMaxPeers];
  unsigned* dep_reset;  // the producer's dependency counter this window resets when it completes (NULL: none)
  unsigned* y16_max;
  const unsigned* x16_max;
  unsigned* clr_max;
  int clr_n;
  float* xsig;          // x-prep launches (x16 given by launch_xprep): 2^σ per (group, batch row) [G][B]
  // L2 prefetch of the next window's weight records (stack graphs, options().l2_prefetch): weights do not depend
  // on activations, so while this window finishes (its tail, the next window's dependency wait and x staging)
  // HBM keeps streaming the next window's records into L2.  CTA c prefetches next-window items c, c + grid, ...
  // (at most pf_items of them; item = one row block's records, contiguous), issued by the producer warp once
  // its own ring is fully issued (pf_at_start = 0) or by its spare lanes at kernel start (1).
  int pf_items;
  int pf_at_start;
  int pf_nm;
  const uint8_t* pf_rec[kMaxMembers];
  int pf_rb_end[kMaxMembers];   // cumulative item counts of the next window's members
  unsigned pf_item_bytes;       // G_next · rec_bytes(bits_next)
  long long* tacc;      // [n_chunks][16 batch][16 ranks][4 tiers] t = V·x in tiered fixed point (self-resetting)
  unsigned* cnt;        // [0] v_done (tile warps done with their V share), [1] w_done (row blocks)
};

// Launch the fused window kernel; bits in {2,3,4}; 1 <= B <= 16.
cudaError_t launch_decode(const DArgs& a, int bits, int grid, cudaStream_t st);
// Whether a launch with this batch / K stages x in shared memory (else it needs launch_xprep first).
bool decode_stages_x(int B, int K);
// Whether an unstaged-x' launch (x16 not given) of this shape runs the int8 path (decode_i8.cuh); such
// a window reads bf16 x itself, so its producer writes no x' hand-off for it.
bool decode_uses_i8(int bits, int B, int K);
// x' (fp16, pre-scaled per the code layout of `bits`) for a !XS decode launch.
cudaError_t launch_xprep(const uint16_t* x, int ldx, int B, int K, int bits, uint16_t* x16, float* xsig, cudaStream_t st,
                         const unsigned* dep_cnt = nullptr, unsigned dep_target = 0);
// Peer mode: wait until this rank's gather counter reaches `target` (system scope), then copy the gathered
// [B][n] bf16 activations to `out` (the stack's final output).
cudaError_t launch_peer_wait_copy(const unsigned* cnt, unsigned target, unsigned* reset, const uint16_t* src, uint16_t* out,
                                  size_t n_elems, cudaStream_t st);
cudaError_t decode_set_trace(void* buf);   // dev: [slots][grid][8] globaltimer stamps (HC_DEC_TRACE builds)
// Max co-resident CTAs of the decode kernel on this device (persistent grid size).
int decode_max_ctas(int bits, int B, int K, int n_chunks, int fwd_chunks, bool no_xs = false);

}  // namespace hc
