/* hcinfer.h — C-ABI of the B200-native HCInfer compensated quantized linear.
 *
 * The library evaluates, per weight matrix, the error-compensated quantized linear of
 * HCInfer (arXiv 2605.05819), §4.1:
 *
 *     y = deq(W_q)·x + U[:, :r]·(V[:r, :]·x),     deq(W_q)[n,k] = s[n,k/g]·(q[n,k] − z[n,k/g])
 *
 * at the rank r chosen by the sensitivity-aware dynamic rank allocation of §4.3 /
 * Appendix B.1.  Matrices that share an input run as one
 * "compensation window" launch (App. A.1.3): QKV, O, UPGATE, DOWN.
 *
 * Conventions (all entry points):
 *   - Every function returns an hc_status; no C++ exception crosses the ABI.  On error
 *     hc_last_error() returns a thread-local, NUL-terminated message (valid until the
 *     next call on that thread).  Status codes mirror SPEC S:713 exit codes.
 *   - "device" pointers are CUDA global-memory pointers on the context's device.
 *     "stream" is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Layouts are row-major, little-endian.  bf16 values travel as uint16 bit patterns.
 *   - There is no CPU fallback: every compute entry point runs hand-written sm_100a
 *     kernels and fails with HC_ERR_RUNTIME when no suitable GPU is present.
 */
#ifndef HCINFER_H
#define HCINFER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HC_OK = 0,
  HC_ERR_CONFIG = 2,   /* invalid argument / shape / bit width / rank */
  HC_ERR_STATE = 3,    /* unknown layer/window, use before load, missing communicator    */
  HC_ERR_NUMERIC = 4,  /* non-finite or negative sensitivity, non-normalised gates */
  HC_ERR_RUNTIME = 5   /* CUDA / NCCL failure, no sm_100 device                            */
} hc_status;

typedef enum { HC_WIN_QKV = 0, HC_WIN_O = 1, HC_WIN_UPGATE = 2, HC_WIN_DOWN = 3 } hc_window_kind;
typedef enum { HC_OUT_F32 = 0, HC_OUT_BF16 = 1 } hc_out_dtype;
typedef enum { HC_GLUE_NONE = 0, HC_GLUE_SILU_MUL = 1 } hc_glue;
typedef enum { HC_FACTORS_BF16 = 0, HC_FACTORS_FP8 = 1 } hc_factor_dtype;

const char* hc_version(void);
const char* hc_last_error(void);

/* =====================================================================================
 * Rank allocation (host only, pure, deterministic, re-entrant).  PAPER.md App. B.1.
 * ===================================================================================== */

/* One weight matrix's allocation inputs.  Windows are keyed by (layer, window_kind);
 * sums over a window run over its members in the order they appear in the array. */
typedef struct {
  int32_t layer;          /* 0 <= layer < budget->n_layers                                 */
  int32_t window_kind;    /* hc_window_kind                                                */
  int32_t slot;           /* member slot inside the window (q,k,v | o | up,gate | down)     */
  int32_t expert;         /* MoE expert id, -1 for dense                                   */
  int32_t n_sigma;        /* length of sigma, or 0                                         */
  const double* sigma;    /* singular values of ΔW, non-increasing; NULL -> use phi */
  double phi;             /* salience φ_i when sigma == NULL                               */
  int32_t n_salient;      /* |S_i| when sigma == NULL (two_stage_mode 1 only)              */
  int32_t n_total;        /* |S_i| + |R_i| when sigma == NULL                              */
  double D_matrix;        /* D_i = KL(P || Q_i) >= 0, an input                 */
  double gate;            /* routing weight g_e of this expert (MoE), else ignored         */
} hc_sens;

typedef struct {
  int32_t n_layers;
  const double* D_layer;  /* [n_layers], D_ℓ >= 0                             */
  int32_t top_k_layers;   /* K of the top-K layer set 𝒯, 1 <= K <= n_layers       */
  double tau;             /* salience threshold τ (0.01)                            */
  int32_t k0;             /* minimum non-zero rank 2^k0 (8 => k0 = 3)           */
  double r_std[4];        /* per-window-kind standard rank r_std, the budget  */
  int32_t two_stage_mode; /* 0: per-matrix reading; 1: pooled literal reading      */
  int32_t moe_k;          /* activated experts per MoE window (𝒢 = k·g_e); 0 = dense */
} hc_budget;

/* φ -> 𝒱 = Norm_W(φ) -> 𝒮_i = Norm_W(D) -> 𝒮_ℓ
 * -> 𝒫 = 𝒢·Norm_W(𝒱𝒮)·𝒮_ℓ -> r̃ = 𝒫·r_std -> two-stage
 * -> Align to {0} ∪ {2^k : k >= k0}, nearest, ties up
 * -> cap: largest level <= caps[i] (R15)
 * -> enforce Σ_W r <= r_std by demoting the lowest-𝒫 member one level (R16).
 * caps[n]: per-matrix maximum rank (min(N, K, r_stored) typically).
 * ranks_out[n]: result.  priority_out[n] (nullable): 𝒫_i.
 * Errors: HC_ERR_CONFIG (bad layer/window/K/k0/n), HC_ERR_NUMERIC (non-finite or
 * negative D, gates of a slot not summing to 1 within 1e-9).  Bit-exact with oracle/allocate.py. */
hc_status hc_allocate_ranks(const hc_sens* recs, int32_t n, const hc_budget* budget,
                            const int32_t* caps, int32_t* ranks_out, double* priority_out);

/* =====================================================================================
 * Context and weights
 * ===================================================================================== */
typedef struct hc_ctx hc_ctx;

/* Create a context on CUDA device `device` (must be sm_100).  *out receives the handle. */
hc_status hc_create(hc_ctx** out, int32_t device);
hc_status hc_destroy(hc_ctx* ctx);

/* One weight matrix in canonical formats (device or host pointers; read during the call only).
 *   codes  uint32 [N][K*bits/32]: row n is a little-endian bitstream, element k at bits
 *          [bits*k, bits*k+bits) — unsigned codes q in [0, 2^bits)            (R1)
 *   scales bf16   [N][K/group]                                                 (R2: groups run along K)
 *   zeros  uint8  [N][K/group], 0 <= z < 2^bits (symmetric RTN: z = 2^(bits-1)) (R3)
 *   U      bf16   [N][r_stored]   (U[:, :r] is the rank-r slice; NULL iff r_stored == 0)
 *   V      bf16   [r_stored][K]   (V[:r, :] is the rank-r slice; absorbs Σ)
 * bits in {2, 3, 4}; group == 128; K % 128 == 0; N % 16 == 0; r_stored % 16 == 0, <= 256;
 * r_alloc in {0} ∪ {8, 16, 32, ...}, r_alloc <= min(r_stored, N, K).
 * row_begin/row_end: the rows [row_begin, row_end) this context keeps (column sharding of
 * the output across GPUs); use 0 / N for an unsharded matrix.
 * (row_end - row_begin) % 16 == 0.
 * factor_dtype: HC_FACTORS_BF16 (U, V as above) or HC_FACTORS_FP8: U and V are e4m3 bytes
 * (uint8 [N][r_stored] and [r_stored][K]; NaN encodings 0x7F / 0xFF rejected with HC_ERR_NUMERIC) with fp32
 * per-rank scales u_scale [r_stored], v_scale [r_stored] (host or device):
 *   U_eff[n][j] = e4m3(U[n][j])·u_scale[j],   V_eff[j][k] = e4m3(V[j][k])·v_scale[j]
 * and the window computes y = deq(W)·x + U_eff[:, :r]·(V_eff[:r, :]·x): half the factor bytes of bf16.  Decode
 * windows read the e4m3 bytes (converted exactly in registers); the prefill path uses fp16 copies of
 * U_eff / V_eff (one fp16 rounding).  Members of a window share the factor dtype; MoE expert windows and
 * t forwarding take bf16 factors only (HC_ERR_CONFIG for fp8 experts).  u_scale / v_scale ignored for bf16.
 * glue: HC_GLUE_SILU_MUL fuses the FFN gate (App. A.1.3, "h = σ(W_gate X) ⊙ W_up X", σ = SiLU)
 * into an UPGATE window: slot 0 = up and slot 1 = gate, same shape, loaded in the SAME call, both
 * flagged; their rows are interleaved at load time (8 up + 8 gate rows per row block) so the
 * window outputs m = silu(gate·x) ⊙ (up·x) (each product compensated at its own rank), width N.
 * Otherwise HC_GLUE_NONE. */
typedef struct {
  int32_t layer, window_kind, slot, expert;
  int32_t N, K, bits, group;
  const uint32_t* codes;
  const uint16_t* scales;
  const uint8_t* zeros;
  const uint16_t* U;
  const uint16_t* V;
  int32_t r_stored, r_alloc;
  int32_t row_begin, row_end;
  int32_t glue;
  int32_t factor_dtype;     /* hc_factor_dtype */
  const float* u_scale;     /* HC_FACTORS_FP8: [r_stored] */
  const float* v_scale;     /* HC_FACTORS_FP8: [r_stored] */
} hc_matrix_desc;

/* Copy + repack matrices into context-owned device memory (synchronous w.r.t. its inputs:
 * the caller may free them on return).  Matrices with equal (layer, window_kind, expert)
 * form one window; members are ordered by `slot`.  Loading a slot again replaces it.
 * Errors: HC_ERR_CONFIG on any shape/bit-width/rank violation. */
hc_status hc_load_layer(hc_ctx* ctx, const hc_matrix_desc* mats, int32_t n_mats, void* stream);

/* Change the allocated rank of one loaded matrix (0 disables its compensation; the
 * r = 0 launch reads no U/V bytes).  HC_ERR_CONFIG if not admissible or > its cap. */
hc_status hc_set_rank(hc_ctx* ctx, int32_t layer, int32_t window_kind, int32_t slot,
                      int32_t expert, int32_t r_alloc);

/* Sum of window output widths (Σ local rows of its members), or -1 if unknown. */
int64_t hc_window_rows(hc_ctx* ctx, int32_t layer, int32_t window_kind, int32_t expert);

/* =====================================================================================
 * Execution (asynchronous on `stream`; caller keeps x / y alive until the stream is done)
 *
 * Concurrency: a context owns per-window workspaces (t accumulators, completion counters, x' hand-off and
 * staging buffers, stack graphs) that every launch resets before it completes.  Launches that use the same
 * window — directly or through hc_stack_forward / hc_moe_forward — must therefore be stream-ordered: calling
 * them concurrently on different streams (or from different host threads) races on those workspaces.  Use
 * one context per concurrent stream.  Different contexts are independent.
 * ===================================================================================== */

/* y[b, :] = concat over the window's members of  deq(W_m)·x_b + U_m[:, :r_m]·(V_m[:r_m, :]·x_b)
 *   x: bf16 [B][K];  y: [B][rows] (fp32 if y_dtype == HC_OUT_F32, else bf16 = RNE of the fp32
 *   value); rows = hc_window_rows(...).  1 <= B <= 16 runs the fused decode kernel.
 *   x and y may be host pointers (pinned or pageable): they are then staged through
 *   context-owned device buffers inside the call (stream-ordered, the call synchronises
 *   the stream before returning). */
hc_status hc_compensated_linear(hc_ctx* ctx, int32_t layer, int32_t window_kind, int32_t expert,
                                const void* x, int32_t B, void* y, int32_t y_dtype, void* stream);

/* Decode step through every loaded dense layer 0..L-1 (R9):
 *   a  = q-part of QKV(h)          (attention is out of scope: identity stand-in on q)
 *   h1 = bf16(h + O(a))            (residual fused into the O epilogue)
 *   m  = bf16(silu(gate) ⊙ up)     (UPGATE loaded with HC_GLUE_SILU_MUL)
 *   h' = bf16(h1 + DOWN(m))        (residual fused into the DOWN epilogue)
 * x: bf16 [B][d] (input hidden state), y: bf16 [B][d] (output of the last layer), 1 <= B <= 16.
 * Every window is one fused decode launch (4 per layer) with programmatic dependent launch; the
 * whole stack is captured once per (B, x, y) into a CUDA graph owned by the context and replayed
 * (re-captured after hc_load_layer / hc_set_rank).  Host x / y are staged like hc_compensated_linear.
 * HC_ERR_STATE if a layer lacks a window or its UPGATE window is not SiLU-fused. */
hc_status hc_stack_forward(hc_ctx* ctx, const void* x, int32_t B, void* y, void* stream);

/* Grouped MoE expert layer (C3; "Y_MoE = Σ_e g_e E_e(X)"):
 *   y[t, :] = Σ_{j<topk} topk_gate[t, j] · DOWN_e(m),  m = bf16(silu(GATE_e(x_t)) ⊙ UP_e(x_t)),
 *   e = topk_idx[t, j], every product compensated at its own rank.
 * The layer's experts are windows (layer, HC_WIN_UPGATE, e) loaded with HC_GLUE_SILU_MUL (slot 0 up,
 * slot 1 gate) and (layer, HC_WIN_DOWN, e) for e = 0 .. E-1 (E = first missing id); all experts share
 * shapes and bits and are unsharded.  x: bf16 [T][K]; topk_idx: int32 [T][topk] (ids outside
 * [0, E) are skipped); topk_gate: fp32 [T][topk] (used as given); y: fp32 [T][D].  1 <= T <= 1024,
 * 1 <= topk <= 16.  One launch per stage over all activated experts: route (group the T·topk
 * (token, expert) rows by expert, tokens ascending), gather + pre-scale x, rank projection
 * t = V·x, grouped compensated GEMV (UPGATE with the SiLU glue), the same for DOWN, combine in slot
 * order.  Deterministic.  Host pointers are staged (the call then synchronises the stream).
 * HC_ERR_STATE if expert 0 is missing or a window is not shaped as above. */
hc_status hc_moe_forward(hc_ctx* ctx, int32_t layer, const void* x, int32_t T, const int32_t* topk_idx,
                         const float* topk_gate, int32_t topk, void* y, void* stream);

/* Dynamic per-(token, expert) compensation ranks for the MoE layer `layer` (P:255-258, P:652-665:
 * the expert activation score G = k·g_e scales the continuous rank): for a routed (token, slot) pair
 * with expert e and gate g, matrix s in (up, gate, down) uses
 *   r = Cap(Align((k·g)·rtilde[3e + s]))   (Align: nearest of {0} ∪ {2^j, j >= k0}, ties up; Cap: the
 *                                            largest level <= the matrix's loaded r_alloc; the product is
 *                                            taken in float64, where it is exact for fp32 g and r̃)
 * instead of its static r_alloc (which stays the upper bound: U / V reads are sized by it).
 * rtilde: host float [n_experts][3] (>= 0, finite), copied; NULL switches back to the static ranks.
 * n_experts must match the layer's experts at the next hc_moe_forward (HC_ERR_CONFIG otherwise).
 * HC_ERR_NUMERIC for a negative or non-finite r̃. */
hc_status hc_moe_set_dynamic_ranks(hc_ctx* ctx, int32_t layer, const float* rtilde, int32_t n_experts, int32_t k0);

/* The per-(token, slot) ranks the device decided in the most recent hc_moe_forward that ran with dynamic
 * ranks (test / inspection export; synchronises the device).  out: host int32 [T][topk][3] = the ranks
 * used for (up, gate, down) of token t's slot j, or -1 for a slot whose expert id was skipped.  T and topk
 * must equal the last call's.  HC_ERR_STATE if that call used static ranks. */
hc_status hc_moe_last_ranks(hc_ctx* ctx, int32_t* out, int32_t T, int32_t topk);

/* Column sharding across GPUs.  Rank 0 calls hc_nccl_unique_id and shares the 128
 * bytes with every rank (e.g. through torch.distributed); each rank then calls hc_set_comm with its
 * rank and the world size (ncclCommInitRank on the context's device; NCCL is loaded at run time).
 * With a communicator set, every member of the stack must hold rows [rank·N/G, (rank+1)·N/G) and
 * hc_stack_forward gathers each window's output slices with ncclAllGather over NVLink before the
 * next window (x and V·x stay replicated).  HC_ERR_RUNTIME if NCCL is unavailable. */
hc_status hc_nccl_unique_id(uint8_t* out128);
hc_status hc_set_comm(hc_ctx* ctx, const uint8_t* id128, int32_t rank, int32_t world);

/* =====================================================================================
 * Calibration (offline, on the GPU).  Produces the compensation factors and the
 * allocator's spectrum input; not on the decode hot path.
 * ===================================================================================== */

/* Factors of the quantization error: ΔW = W − deq(codes, scales, zeros) in float64
 * (deq as hcinfer.h's canonical formats, R1-R3), its SVD ΔW = P·diag(σ)·Qᵀ by one-sided Jacobi in
 * float64 (the shorter side of ΔW is orthogonalised; fixed-order reductions, deterministic), and
 *   U = P[:, :r]  (float64 [n_mats][N][r]),   V = diag(σ[:r])·Q[:, :r]ᵀ  (float64 [n_mats][r][K])   (R4)
 * with the sign convention "first nonzero entry of each U column >= 0" (R5); sigma (float64 [n_mats][min(N,K)],
 * non-increasing) if non-NULL.  Batched over n_mats matrices of one shape.  All pointers device memory;
 * W float32 [n_mats][N][K] (the unquantized weights), codes / scales / zeros canonical [n_mats][N][...].
 * N, K multiples of 32; group divides K; bits in {2, 3, 4, 8}; 0 <= r <= min(N, K).  sweeps_out (host,
 * nullable): Jacobi sweeps run.  Synchronises the stream (the convergence test reads a device word per
 * sweep).  Workspace: context-owned, about 16·N·K·n_mats bytes.  HC_ERR_CONFIG on bad shapes or
 * pointers. */
hc_status hc_calib_svd(hc_ctx* ctx, const float* W, const uint32_t* codes, const uint16_t* scales, const uint8_t* zeros,
                       int32_t n_mats, int32_t N, int32_t K, int32_t bits, int32_t group, int32_t r,
                       double* U_out, double* V_out, double* sigma_out, int32_t* sweeps_out, void* stream);

/* Salience φ of each spectrum (App. B.1 eq. A8, R10) on the device: σ̂ = σ/σ₁,
 * k_j = σ̂_{j−1} − 2σ̂_j + σ̂_{j+1} over interior j, cut = argmax (smallest index on ties), S = {1..cut} iff
 * max k > tau, φ = mean_S σ / max(mean_R σ, 1e-300), else φ = 1 (n < 3 or σ₁ = 0: φ = 1).  sigma: device
 * float64 [n_mats][n]; phi_out device float64 [n_mats]; n_salient_out device int32 [n_mats] (|S|, 0 if ∅).
 * The float64 operations of oracle/allocate.py salience in its order (no contraction): bit-exact given σ. */
hc_status hc_calib_salience(hc_ctx* ctx, const double* sigma, int32_t n_mats, int32_t n, double tau,
                            double* phi_out, int32_t* n_salient_out, void* stream);

/* B200 budget r_std of a compensation window (R17, the analogue of P:278-289's CPU-time budget):
 * the largest rank whose factor bytes stay within eps of the window's base bytes,
 *   r_std = floor(eps · bytes_base / (2·(N̄ + K))),  bytes_base = Σ_i N_i·K·bits/8 + N_i·(K/group)·(16 + bits)/8,
 * N̄ = mean N_i (eps = 0.1 for the ≤10% target).  Host only, pure. */
hc_status hc_calib_r_std(const int32_t* Ns, int32_t n_members, int32_t K, int32_t bits, int32_t group, double eps,
                         double* r_std_out);

/* Process-wide development switches, for A/B timing of equivalent plans (every setting computes the same
 * product up to fp32 accumulation order; the parity tests pass under each).  Read when a window plan or a
 * stack graph is built; setting one makes contexts re-capture their stack graphs on the next call.
 *   "t_forward"          0  stack: window w-1's epilogue accumulates window w's t = V·x
 *   "x_handoff"          1  stack: the producer epilogue writes the next fp16-path window's x' (§7.1)
 *   "dep_wait"           1  stack: wait on the producer window's counter, not the kernel boundary (§7.1)
 *   "int8_path"          1  decode: u8·s8 tensor-core path for 2-/4-bit codes at B <= 2 (§7.1)
 *   "prefill_merge"      1  prefill: one GEMM over a multi-member window (§7.5)
 *   "decode_ctas_per_sm" 0  decode: cap on resident CTAs per SM (0 = the occupancy limit)
 *   "pdl"                1  decode: programmatic dependent launch between consecutive windows
 *   "l2_prefetch"        0  stack: next-window record items each CTA prefetches into L2 (0 = off)
 *   "l2_prefetch_at_start" 0  stack: issue those prefetches at kernel start instead of after the CTA's own ring
 * HC_ERR_CONFIG for an unknown name or a negative value.  Not thread-safe against concurrent launches. */
hc_status hc_set_option(const char* name, int32_t value);
hc_status hc_get_option(const char* name, int32_t* value);

/* Peer mode: the column-sharded stack with the gather FUSED into the decode epilogue.
 * Every window's epilogue stores its output rows into the full-width activation buffer of every rank (peer
 * memory over NVLink / NVSwitch), adds the next window's t partials of its own output slice
 * (V_next[:, slice]·y_slice) into every rank's t accumulators — so no rank recomputes V·x over the full x —
 * and bumps every rank's gather counter with a system-scope release; the next window waits for G times its
 * producer's rows (system-scope acquire).  No NCCL call, no unshard kernel, one launch per window.  After the
 * last layer one tiny kernel waits for the final gather and copies it to y.
 * Setup, after every rank loaded its shard (rows [rank·N/G, (rank+1)·N/G) of every member):
 *   hc_peer_region(ctx, G, &base, &bytes)   allocates this rank's region (gathered activations, per-window
 *                                          counters and t accumulators; the same layout on every rank)
 *   then EITHER hc_peer_ipc_handle + exchange (e.g. torch.distributed) + hc_peer_connect  (one process per GPU)
 *   OR hc_peer_set with the bases already mapped in this process.
 * Then hc_stack_forward runs the peer graph (priority over hc_set_comm's NCCL path).  Ranks must call
 * hc_stack_forward with the same B and x, concurrently; a rank whose peers never arrive traps after ~20 s
 * (HC_ERR_RUNTIME) instead of hanging.  2 <= G <= 8.  hc_peer_region again after hc_set_rank raises a
 * window's rank beyond the region's t capacity. */
hc_status hc_peer_region(hc_ctx* ctx, int32_t world, void** base_out, uint64_t* bytes_out);
hc_status hc_peer_ipc_handle(hc_ctx* ctx, uint8_t* out64);
hc_status hc_peer_connect(hc_ctx* ctx, int32_t rank, int32_t world, const uint8_t* handles /* [world][64] */);
hc_status hc_peer_set(hc_ctx* ctx, int32_t rank, int32_t world, void* const* bases /* [world] */);

/* Debug/test exports (host only, no GPU needed): the load-time repack and its inverse. */
size_t hc_repacked_bytes(int32_t N, int32_t K, int32_t bits);
hc_status hc_repack_host(const uint32_t* codes, const uint16_t* scales, const uint8_t* zeros,
                         int32_t N, int32_t K, int32_t bits, uint8_t* out);
/* Decode a repacked buffer back to unsigned codes q[N][K], scales bf16 [N][K/128], zeros [N][K/128]
 * through the kernel's own fragment/slot mapping. */
hc_status hc_unpack_repacked_host(const uint8_t* packed, int32_t N, int32_t K, int32_t bits,
                                  uint8_t* q_out, uint16_t* scales_out, uint8_t* zeros_out);
/* The column-sharding gather permutation on the host: all-gathered slices [G][B][n_local] (a window
 * of n_members members with local widths widths[], n_local = Σ widths) -> canonical [B][G·n_local]
 * (member m's full rows are the G local slices in rank order).  Same index map as the device kernel
 * hc_stack_forward uses after ncclAllGather. */
hc_status hc_unshard_host(const uint16_t* gathered, uint16_t* out, int32_t G, int32_t B, int32_t n_members,
                          const int32_t* widths);

#ifdef __cplusplus
}
#endif
#endif /* HCINFER_H */
