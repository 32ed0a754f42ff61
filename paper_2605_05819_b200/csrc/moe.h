// Grouped MoE expert path: one launch per window over all activated experts
// (the paper's cross-expert window fusion).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace hc {

constexpr int kMoEMaxK = 16;            // top-k per token

// One expert's matrices of one window kind, device side (records / U / V layouts of layout.h).
struct MoEExpert {
  const uint8_t* rec;       // [n_rb][G][rec_bytes] (UPGATE: 8 up + 8 gate rows interleaved per row block)
  const uint4* U;           // [n_rb][rs(0)/16][32] bf16 A-fragments (UPGATE: interleaved up/gate rows)
  const uint4* Vn[2];       // natural-k V fragments [K/16][rs/16][32] of member 0 (up | down) and 1 (gate)
  int r[2];                 // allocated ranks (0: no compensation)
  int rs[2];                // r_stored
};

// Routing tables written by moe_route (all device memory, sized for T·k rows and E + T·k entries).
struct MoERoute {
  int* n_rows;      // [1] rows = Σ_e n_e (= T·k)
  int* n_ent;       // [1] grouped entries
  int* row_tok;     // [R] token of each row; rows grouped by expert (ascending), tokens ascending
  int* tok_row;     // [T][k] row of (token, slot)
  int* ent_e;       // [E + R] expert of entry
  int* ent_row0;    // [E + R] first row of entry (entries = chunks of <= 16 rows of one expert)
  int* ent_ncol;    // [E + R] rows in entry
};

struct MoEWin {
  const MoEExpert* ex;      // [E] device
  int n_rb, K, G, glue;     // per expert: row blocks, input width; glue = fused SiLU(gate)·up (UPGATE)
  int t_ld;                 // floats per row of the t buffer (= 2 · max rank chunk · 16)
  const uint16_t* row_rank; // dynamic ranks [R][3] (up, gate, down) per routed row, or NULL (static ranks)
  int rank_slot0;           // slot of member 0 in row_rank: 0 (UPGATE: up, gate), 2 (DOWN)
};

// Dynamic per-(token, expert) ranks: r = Cap(Align((k·g)·r̃[e][s])), decided in
// float64 (exact for fp32 g and r̃); rtilde / caps are [E][3] (up, gate, down), k0 the smallest nonzero
// level exponent.
struct MoEDyn {
  const float* rtilde;
  const int* caps;
  int k0;
  uint16_t* row_rank;       // out: [R][3]
};

// Route: group (token, slot) pairs by expert (deterministic order), build entries of <= 16 rows.
cudaError_t moe_route(const int32_t* topk_idx, const float* topk_gate, int T, int k, int E, const MoERoute& rt,
                      const MoEDyn* dyn, cudaStream_t st);
// x rows of every routed (token, expert) row: xg = x[row_tok] (bf16) and x16 = x'(bits) (fp16).
// gather == 0: the rows are x itself (row r = row r, used for the DOWN input m).
// xsig: [R][K/128] the per-(row, group) factors 2^σ of the x' prescale (R20).
cudaError_t moe_prep(const uint16_t* x, int ldx, int K, int bits, int gather, const MoERoute& rt, int R_max,
                     uint16_t* xg, uint16_t* x16, float* xsig, cudaStream_t st);
// t[row][m][rank] = V_m·x_row for every row of every entry (members m < 1 + glue), fp32.
cudaError_t moe_rank_proj(const MoEWin& w, const MoERoute& rt, int max_ent, const uint16_t* xg, float* t,
                          cudaStream_t st);
// Grouped compensated GEMV: out rows of every entry.  glue: out = bf16 m [R][n_rb·8];
// else out = fp32 [R][n_rb·16].
// max_cols: an upper bound on the rows of an entry (min(T, 16)): <= 8 selects the 8-column mma variant.
cudaError_t moe_gemv(const MoEWin& w, int bits, const MoERoute& rt, int max_ent, const uint16_t* x16,
                     const float* xsig, const float* t, void* out, int max_cols, cudaStream_t st);
// y[t][n] = Σ_j g[t][j] · dout[tok_row[t][j]][n]   (fixed slot order)
cudaError_t moe_combine(const float* dout, int N, const float* topk_gate, int T, int k, const MoERoute& rt,
                        float* y, cudaStream_t st);

}  // namespace hc
