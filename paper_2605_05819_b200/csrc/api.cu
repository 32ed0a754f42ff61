// C-ABI: context, load_layer (copy + repack), set_rank, compensated_linear, stack_forward (hcinfer.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "calib.h"
#include "comm.h"
#include "options.h"
#include "decode.h"
#include "prefill.h"
#include "moe.h"
#include "hcinfer.h"
#include "layout.h"
#include "repack_kernels.h"
#include "status.h"

using hc::fail;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t n) {
    if (p) { cudaFree(p); p = nullptr; }
    bytes = n;
    return n ? cudaMalloc(&p, n) : cudaSuccess;
  }
};

struct Member {
  int slot = 0, N = 0, K = 0, bits = 0, r_stored = 0, r_alloc = 0, row_begin = 0, row_end = 0;
  std::shared_ptr<DevBuf> rec, U, V;   // rec/U empty for the gate member of a fused SiLU window
  std::shared_ptr<DevBuf> Vn;          // natural-k V fragments [K/16][r_stored/16][32] (t forwarding)
  // prefill (tcgen05) copies, 4-bit plain members only: nibble-paired codes, canonical scales /
  // zeros of the shard rows, fp16 U [rows][r_stored] and V [r_stored][K]
  std::shared_ptr<DevBuf> pcodes, pscales, pzeros, U16, V16;
  bool fp8 = false;                    // e4m3 factors (U / V hold U8 / V8 fragments) with per-rank scales us / vs
  std::shared_ptr<DevBuf> us, vs;      // fp32 [r_stored]
  int rows() const { return row_end - row_begin; }
  int cap() const { return std::min(std::min(r_stored, N), K); }
};

// Prefill copies of a multi-member window merged into one GEMM (rows concatenated, rank slices
// stacked: T = X·[V_0[:r_0]; V_1[:r_1]; ...]ᵀ and a block-diagonal U), rebuilt when ranks change.
struct PrefillMerged {
  DevBuf codes, scales, zeros, V, U;
  std::vector<int> ranks;      // r_alloc of each member the buffers were built for
  int R = 0;                   // Σ ceil16(r_i)
  bool valid = false;
};

struct Window {
  int layer = 0, kind = 0, expert = -1;
  std::shared_ptr<PrefillMerged> pm = std::make_shared<PrefillMerged>();
  int glue = HC_GLUE_NONE;            // SILU_MUL: members[0] = up (interleaved records), [1] = gate
  std::vector<Member> members;        // sorted by slot
  DevBuf tacc, cnt;                   // launch workspace: fixed-point t, counters (self-resetting)
  DevBuf xprep;                       // !XS launches: fp16 x' [16][K]
  int ws_chunks = -1;
  int64_t out_rows() const {
    if (glue == HC_GLUE_SILU_MUL) return members.front().rows();
    int64_t n = 0;
    for (const Member& m : members) n += m.rows();
    return n;
  }
};

using Key = std::tuple<int, int, int>;

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

bool admissible_rank(int r) { return r == 0 || (r >= 8 && (r & (r - 1)) == 0); }

struct StackGraph {
  cudaGraphExec_t exec = nullptr;
  unsigned epoch = 0;                 // options().epoch at capture
  ~StackGraph() { if (exec) cudaGraphExecDestroy(exec); }
};

}  // namespace

struct hc_ctx {
  int device = 0;
  int sms = 0;
  std::map<Key, Window> windows;
  std::map<std::tuple<int, int, int, int, int>, int> max_ctas;   // (bits, B, K, chunks, vks) -> co-resident CTAs
  DevBuf stage_x, stage_y;
  DevBuf p_x16, p_t16, p_tpart, p_rsig;        // prefill scratch: fp16 activations, fp16 T = X·Vᵀ, split-K partials
  // decode stack (hc_stack_forward)
  DevBuf s_h, s_h1, s_qkv, s_m;
  int trace_slot = 0;                  // dev tracing: slot of the next decode launch (HC_DEC_TRACE builds)
  DevBuf s_x16[4];                     // x' hand-off buffers of the stack: q, h1, m, h (16 rows each)
  DevBuf s_x16max;                     // their per-(group, batch row) max |x| [4][G][16] (DArgs::y16_max / x16_max)
  std::map<std::tuple<int, const void*, void*>, std::unique_ptr<StackGraph>> graphs;
  cudaStream_t cap_stream = nullptr;
  // column sharding (hc_set_comm): NCCL communicator, send / gather staging
  hc::Comm* comm = nullptr;
  int rank = 0, world = 1;
  DevBuf t_send, t_gather;
  // grouped MoE (hc_moe_forward): per-layer device expert tables, rebuilt after load / set_rank
  struct MoECache {
    DevBuf ex_ug, ex_dn;
    int E = 0, K = 0, F = 0, D = 0, bits = 0, t_ug = 32, t_dn = 32;
    bool valid = false;
    // dynamic per-(token, expert) ranks (hc_moe_set_dynamic_ranks): host r̃ [E][3], device r̃ and caps
    std::vector<float> rtilde;
    int k0 = 3;
    DevBuf d_rtilde, d_caps;
  };
  std::map<int, MoECache> moe;
  DevBuf moe_ws, moe_idx, moe_gate;
  DevBuf calib_ws;                     // hc_calib_svd workspace
  // peer mode (hc_peer_region / hc_peer_set / hc_peer_connect): column-sharded stack with the gather fused
  // into the decode epilogue over peer memory.  The region has the same layout on every
  // rank: the four gathered activations, then per window a gather counter and the t accumulators.
  struct Peer {
    bool on = false;
    DevBuf region;
    void* base[hc::kMaxPeers] = {};    // every rank's region mapped in this process (own included)
    std::vector<void*> opened;         // IPC mappings to close
    size_t off_qkv = 0, off_h1 = 0, off_m = 0, off_h = 0, off_win = 0, win_stride = 0, bytes = 0;
    int n_win = 0, G = 0, mc = 0;
  } peer;
  // the last hc_moe_forward with dynamic ranks (hc_moe_last_ranks): routing shape and device tables
  struct { int T = 0, topk = 0; const int* tok_row = nullptr; const uint16_t* row_rank = nullptr; } moe_last;
  void invalidate_graphs() {
    graphs.clear();
    for (auto& kv : windows) kv.second.pm->valid = false;
    for (auto& kv : moe) kv.second.valid = false;
  }
};

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) return fail(HC_ERR_RUNTIME, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

extern "C" const char* hc_version(void) { return "hcinfer-b200 0.2 (sm_100a)"; }
extern "C" const char* hc_last_error(void) { return hc::last_error_buf(); }

extern "C" hc_status hc_create(hc_ctx** out, int32_t device) {
  if (!out) return fail(HC_ERR_CONFIG, "hc_create: out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) { cudaGetLastError(); return fail(HC_ERR_RUNTIME, "hc_create: no CUDA device (%s)", cudaGetErrorString(e)); }
  if (device < 0 || device >= n) return fail(HC_ERR_CONFIG, "hc_create: device %d out of range [0, %d)", device, n);
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10 || prop.minor != 0)
    return fail(HC_ERR_RUNTIME, "hc_create: device %d is sm_%d%d; this library is built for sm_100a only", device, prop.major, prop.minor);
  CUDA_TRY(cudaSetDevice(device));
  hc_ctx* c = new hc_ctx();
  c->device = device;
  c->sms = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(HC_ERR_RUNTIME, "hc_create: stream creation failed");
  }
  *out = c;
  return HC_OK;
}

extern "C" hc_status hc_destroy(hc_ctx* ctx) {
  if (!ctx) return HC_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  ctx->graphs.clear();
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  hc::comm_destroy(ctx->comm);
  for (void* p : ctx->peer.opened) cudaIpcCloseMemHandle(p);
  delete ctx;
  return HC_OK;
}

extern "C" hc_status hc_nccl_unique_id(uint8_t* out) {
  if (!out) return fail(HC_ERR_CONFIG, "hc_nccl_unique_id: null output");
  char msg[256];
  if (!hc::comm_unique_id(out, msg, sizeof(msg))) return fail(HC_ERR_RUNTIME, "%s", msg);
  return HC_OK;
}

extern "C" hc_status hc_set_comm(hc_ctx* ctx, const uint8_t* id, int32_t rank, int32_t world) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_set_comm: null context");
  if (!id || world < 1 || rank < 0 || rank >= world) return fail(HC_ERR_CONFIG, "hc_set_comm: rank %d / world %d", rank, world);
  CUDA_TRY(cudaSetDevice(ctx->device));
  char msg[256];
  hc::Comm* c = hc::comm_create(id, rank, world, msg, sizeof(msg));
  if (!c) return fail(HC_ERR_RUNTIME, "%s", msg);
  hc::comm_destroy(ctx->comm);
  ctx->comm = c;
  ctx->rank = rank;
  ctx->world = world;
  ctx->invalidate_graphs();
  return HC_OK;
}

static hc_status validate_desc(const hc_matrix_desc& d, int i) {
  if (d.window_kind < 0 || d.window_kind > 3) return fail(HC_ERR_CONFIG, "mat %d: window_kind %d", i, d.window_kind);
  if (d.bits != 2 && d.bits != 3 && d.bits != 4) return fail(HC_ERR_CONFIG, "mat %d: bits %d not in {2,3,4}", i, d.bits);
  if (d.group != hc::kGroup) return fail(HC_ERR_CONFIG, "mat %d: group %d != 128", i, d.group);
  if (d.K <= 0 || d.K % hc::kGroup) return fail(HC_ERR_CONFIG, "mat %d: K %d not a multiple of 128", i, d.K);
  if (d.N <= 0 || d.N % hc::kRows) return fail(HC_ERR_CONFIG, "mat %d: N %d not a multiple of 16", i, d.N);
  if (d.row_begin < 0 || d.row_end > d.N || d.row_end <= d.row_begin || (d.row_end - d.row_begin) % hc::kRows || d.row_begin % hc::kRows)
    return fail(HC_ERR_CONFIG, "mat %d: shard rows [%d, %d) invalid for N %d (16-row units)", i, d.row_begin, d.row_end, d.N);
  if (d.r_stored < 0 || d.r_stored % 16 || d.r_stored > 256) return fail(HC_ERR_CONFIG, "mat %d: r_stored %d", i, d.r_stored);
  if (!admissible_rank(d.r_alloc) || d.r_alloc > std::min(std::min(d.r_stored, d.N), d.K))
    return fail(HC_ERR_CONFIG, "mat %d: r_alloc %d not admissible or > cap", i, d.r_alloc);
  if (!d.codes || !d.scales || !d.zeros) return fail(HC_ERR_CONFIG, "mat %d: null codes/scales/zeros", i);
  if (d.r_stored > 0 && (!d.U || !d.V)) return fail(HC_ERR_CONFIG, "mat %d: r_stored > 0 needs U and V", i);
  if (d.glue != HC_GLUE_NONE && d.glue != HC_GLUE_SILU_MUL) return fail(HC_ERR_CONFIG, "mat %d: glue %d", i, d.glue);
  if (d.factor_dtype != HC_FACTORS_BF16 && d.factor_dtype != HC_FACTORS_FP8)
    return fail(HC_ERR_CONFIG, "mat %d: factor_dtype %d", i, d.factor_dtype);
  if (d.factor_dtype == HC_FACTORS_FP8 && d.expert >= 0)
    return fail(HC_ERR_CONFIG, "mat %d: fp8 factors are for dense windows (MoE experts take bf16 factors)", i);
  if (d.factor_dtype == HC_FACTORS_FP8 && d.r_stored > 0 && (!d.u_scale || !d.v_scale))
    return fail(HC_ERR_CONFIG, "mat %d: fp8 factors need u_scale and v_scale", i);
  if (d.glue == HC_GLUE_SILU_MUL && (d.window_kind != HC_WIN_UPGATE || (d.slot != 0 && d.slot != 1)))
    return fail(HC_ERR_CONFIG, "mat %d: SiLU glue needs an UPGATE window with slots 0 (up) and 1 (gate)", i);
  return HC_OK;
}

// Canonical (host or device) inputs of one matrix, resident on the device for the repack.
struct Staged {
  DevBuf tc, ts, tz, tu, tv;
  const uint32_t* codes = nullptr;
  const uint16_t* scales = nullptr;
  const uint8_t* zeros = nullptr;
  const uint16_t *U = nullptr, *V = nullptr;     // bf16, or the e4m3 bytes (fp8 factors)
  DevBuf tus, tvs;
  const float *us = nullptr, *vs = nullptr;      // fp8 per-rank scales
};

static const void* to_device(const void* src, size_t bytes, DevBuf& tmp, cudaStream_t st, cudaError_t& err) {
  err = cudaSuccess;
  if (is_device_ptr(src)) return src;
  err = tmp.alloc(bytes);
  if (err != cudaSuccess) return nullptr;
  err = cudaMemcpyAsync(tmp.p, src, bytes, cudaMemcpyHostToDevice, st);
  return tmp.p;
}

static hc_status stage(const hc_matrix_desc& d, Staged& s, cudaStream_t st) {
  const int G = d.K / hc::kGroup;
  cudaError_t e;
  s.codes = (const uint32_t*)to_device(d.codes, (size_t)d.N * d.K * d.bits / 8, s.tc, st, e);
  CUDA_TRY(e);
  s.scales = (const uint16_t*)to_device(d.scales, (size_t)d.N * G * 2, s.ts, st, e);
  CUDA_TRY(e);
  s.zeros = (const uint8_t*)to_device(d.zeros, (size_t)d.N * G, s.tz, st, e);
  CUDA_TRY(e);
  if (d.r_stored > 0) {
    const size_t es = d.factor_dtype == HC_FACTORS_FP8 ? 1 : 2;
    s.U = (const uint16_t*)to_device(d.U, (size_t)d.N * d.r_stored * es, s.tu, st, e);
    CUDA_TRY(e);
    s.V = (const uint16_t*)to_device(d.V, (size_t)d.r_stored * d.K * es, s.tv, st, e);
    CUDA_TRY(e);
    if (d.factor_dtype == HC_FACTORS_FP8) {
      s.us = (const float*)to_device(d.u_scale, (size_t)d.r_stored * 4, s.tus, st, e);
      CUDA_TRY(e);
      s.vs = (const float*)to_device(d.v_scale, (size_t)d.r_stored * 4, s.tvs, st, e);
      CUDA_TRY(e);
    }
  }
  return HC_OK;
}

static Member make_member(const hc_matrix_desc& d) {
  Member m;
  m.slot = d.slot; m.N = d.N; m.K = d.K; m.bits = d.bits; m.r_stored = d.r_stored; m.r_alloc = d.r_alloc;
  m.row_begin = d.row_begin; m.row_end = d.row_end;
  m.rec = std::make_shared<DevBuf>();
  m.U = std::make_shared<DevBuf>();
  m.V = std::make_shared<DevBuf>();
  m.Vn = std::make_shared<DevBuf>();
  m.pcodes = std::make_shared<DevBuf>();
  m.pscales = std::make_shared<DevBuf>();
  m.pzeros = std::make_shared<DevBuf>();
  m.U16 = std::make_shared<DevBuf>();
  m.V16 = std::make_shared<DevBuf>();
  m.fp8 = d.factor_dtype == HC_FACTORS_FP8;
  m.us = std::make_shared<DevBuf>();
  m.vs = std::make_shared<DevBuf>();
  return m;
}

// Prefill copies of a plain 4-bit member, built on the device from its decode records and factor fragments the
// first time a B > 16 launch needs them (a decode-only stack never pays their memory): nibble-paired codes,
// scales / zeros transposed to [G][rows], fp16 U [rows][r_stored] and V [r_stored][K] (fp8 factors: fp16 of
// e4m3 · scale).
static hc_status ensure_prefill(Member& m, cudaStream_t st) {
  if (m.bits != 4 || (m.pcodes && m.pcodes->p)) return HC_OK;
  const int rows = m.rows(), G = m.K / hc::kGroup, wpr = m.K / 8;
  DevBuf q, codes, sc, zr;
  CUDA_TRY(q.alloc((size_t)rows * m.K));
  CUDA_TRY(codes.alloc((size_t)rows * wpr * 4));
  CUDA_TRY(sc.alloc((size_t)rows * G * 2));
  CUDA_TRY(zr.alloc((size_t)rows * G));
  if (m.r_stored > 0) {
    CUDA_TRY(m.U16->alloc((size_t)rows * m.r_stored * 2));
    CUDA_TRY(m.V16->alloc((size_t)m.r_stored * m.K * 2));
  }
  CUDA_TRY(hc::launch_unrepack_prefill((const uint8_t*)m.rec->p, rows / hc::kRows, m.K, m.bits, (uint8_t*)q.p,
                                       (uint32_t*)codes.p, (uint16_t*)sc.p, (uint8_t*)zr.p, (const uint8_t*)m.U->p,
                                       (const uint8_t*)m.V->p, m.r_stored, m.fp8 ? (const float*)m.us->p : nullptr,
                                       m.fp8 ? (const float*)m.vs->p : nullptr, (uint16_t*)m.U16->p, (uint16_t*)m.V16->p, st));
  CUDA_TRY(m.pcodes->alloc((size_t)rows * wpr * 4));
  CUDA_TRY(hc::launch_prefill_codes((const uint32_t*)codes.p, (uint32_t*)m.pcodes->p, (size_t)rows * wpr, st));
  CUDA_TRY(m.pscales->alloc((size_t)rows * G * 2));   // transposed [G][rows]
  CUDA_TRY(m.pzeros->alloc((size_t)rows * G));
  CUDA_TRY(hc::launch_transpose_groups((const uint16_t*)sc.p, (const uint8_t*)zr.p, rows, G, (uint16_t*)m.pscales->p,
                                       (uint8_t*)m.pzeros->p, st));
  CUDA_TRY(cudaStreamSynchronize(st));                // the temporaries die at scope end
  return HC_OK;
}

// fp8 factors of one member (or the fused pair): U8 fragments from rows U0 / U1 (rstride as RepackSrc), V8
// pieces, the per-rank scales copied to member-owned buffers; HC_ERR_NUMERIC on a NaN encoding.
static hc_status load_fp8(Member& m, const uint8_t* U0, const uint8_t* U1, int rstride, int n_rb, const Staged& sd,
                          bool with_u, cudaStream_t st) {
  if (m.r_stored == 0) return HC_OK;
  DevBuf flag;
  CUDA_TRY(flag.alloc(sizeof(unsigned)));
  CUDA_TRY(cudaMemsetAsync(flag.p, 0, sizeof(unsigned), st));
  if (with_u) CUDA_TRY(m.U->alloc((size_t)n_rb * hc::kRows * m.r_stored));
  CUDA_TRY(m.V->alloc((size_t)m.r_stored * m.K));
  CUDA_TRY(hc::launch_repack_fp8(U0, U1, rstride, with_u ? n_rb : 0, (const uint8_t*)sd.V, m.K, m.r_stored,
                                 with_u ? (uint8_t*)m.U->p : nullptr, (uint8_t*)m.V->p, (unsigned*)flag.p, st));
  CUDA_TRY(m.us->alloc((size_t)m.r_stored * 4));
  CUDA_TRY(m.vs->alloc((size_t)m.r_stored * 4));
  CUDA_TRY(cudaMemcpyAsync(m.us->p, sd.us, (size_t)m.r_stored * 4, cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(m.vs->p, sd.vs, (size_t)m.r_stored * 4, cudaMemcpyDeviceToDevice, st));
  unsigned h = 0;
  CUDA_TRY(cudaMemcpyAsync(&h, flag.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (h) return fail(HC_ERR_NUMERIC, "fp8 factors: NaN encoding (0x7F / 0xFF) in U or V");
  std::vector<float> sc(2 * m.r_stored);
  CUDA_TRY(cudaMemcpy(sc.data(), m.us->p, (size_t)m.r_stored * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(sc.data() + m.r_stored, m.vs->p, (size_t)m.r_stored * 4, cudaMemcpyDeviceToHost));
  for (float v : sc)
    if (!std::isfinite(v)) return fail(HC_ERR_NUMERIC, "fp8 factors: non-finite scale");
  return HC_OK;
}

// Load matrix i (and, for a fused SiLU pair, its partner) into its window.  On failure the caller drops a
// window this call created and left empty.
static hc_status load_one(hc_ctx* ctx, const hc_matrix_desc* mats, int32_t n_mats, int i, std::vector<char>& done,
                          cudaStream_t st) {
    const hc_matrix_desc& d = mats[i];
    Key key{d.layer, d.window_kind, d.expert};
    Window& w = ctx->windows[key];
    w.layer = d.layer; w.kind = d.window_kind; w.expert = d.expert;
    const int G = d.K / hc::kGroup;

    if (d.glue == HC_GLUE_SILU_MUL) {
      // ---- fused SiLU(gate)·up window: find the partner in this call, interleave rows 8 + 8
      int j = -1;
      for (int k = 0; k < n_mats; ++k)
        if (k != i && !done[k] && mats[k].glue == HC_GLUE_SILU_MUL && mats[k].layer == d.layer &&
            mats[k].window_kind == d.window_kind && mats[k].expert == d.expert && mats[k].slot != d.slot)
          j = k;
      if (j < 0) return fail(HC_ERR_CONFIG, "mat %d: SiLU glue needs up and gate in the same hc_load_layer call", i);
      const hc_matrix_desc& up = d.slot == 0 ? d : mats[j];
      const hc_matrix_desc& gate = d.slot == 0 ? mats[j] : d;
      if (up.N != gate.N || up.K != gate.K || up.bits != gate.bits || up.r_stored != gate.r_stored ||
          up.row_begin != gate.row_begin || up.row_end != gate.row_end || up.factor_dtype != gate.factor_dtype)
        return fail(HC_ERR_CONFIG, "SiLU glue: up and gate must have identical shape, bits, r_stored, shard and factor dtype");
      const bool f8 = up.factor_dtype == HC_FACTORS_FP8;
      Member mu = make_member(up), mg = make_member(gate);
      const int rows = mu.rows();
      Staged su, sg;
      hc_status s = stage(up, su, st);
      if (s != HC_OK) return s;
      s = stage(gate, sg, st);
      if (s != HC_OK) return s;
      CUDA_TRY(mu.rec->alloc((size_t)(rows / 8) * G * hc::rec_bytes(up.bits)));
      if (up.r_stored > 0 && !f8) {
        CUDA_TRY(mu.U->alloc((size_t)2 * rows * up.r_stored * 2));
        CUDA_TRY(mu.V->alloc((size_t)up.r_stored * up.K * 2));
        CUDA_TRY(mg.V->alloc((size_t)gate.r_stored * gate.K * 2));
      }
      const int wpr = up.K * up.bits / 32;
      hc::RepackSrc src;
      src.codes[0] = su.codes + (size_t)up.row_begin * wpr;  src.codes[1] = sg.codes + (size_t)up.row_begin * wpr;
      src.scales[0] = su.scales + (size_t)up.row_begin * G;  src.scales[1] = sg.scales + (size_t)up.row_begin * G;
      src.zeros[0] = su.zeros + (size_t)up.row_begin * G;    src.zeros[1] = sg.zeros + (size_t)up.row_begin * G;
      src.U[0] = (su.U && !f8) ? su.U + (size_t)up.row_begin * up.r_stored : nullptr;
      src.U[1] = (sg.U && !f8) ? sg.U + (size_t)up.row_begin * up.r_stored : nullptr;
      src.rstride = 8;
      CUDA_TRY(hc::launch_repack_records(src, up.K, up.bits, f8 ? 0 : up.r_stored, rows / 8, (uint8_t*)mu.rec->p,
                                         (uint32_t*)mu.U->p, st));
      if (f8) {
        hc_status s8 = load_fp8(mu, (const uint8_t*)su.U + (size_t)up.row_begin * up.r_stored,
                                (const uint8_t*)sg.U + (size_t)up.row_begin * up.r_stored, 8, rows / 8, su, true, st);
        if (s8 == HC_OK) s8 = load_fp8(mg, nullptr, nullptr, 8, rows / 8, sg, false, st);
        if (s8 != HC_OK) return s8;
      } else {
        CUDA_TRY(hc::launch_repack_v(su.V, up.K, up.r_stored, (uint32_t*)mu.V->p, st));
        CUDA_TRY(hc::launch_repack_v(sg.V, gate.K, gate.r_stored, (uint32_t*)mg.V->p, st));
      }
      if (up.r_stored > 0 && !f8) {
        CUDA_TRY(mu.Vn->alloc((size_t)up.r_stored * up.K * 2));
        CUDA_TRY(mg.Vn->alloc((size_t)gate.r_stored * gate.K * 2));
        CUDA_TRY(hc::launch_repack_vn(su.V, up.K, up.r_stored, (uint32_t*)mu.Vn->p, st));
        CUDA_TRY(hc::launch_repack_vn(sg.V, gate.K, gate.r_stored, (uint32_t*)mg.Vn->p, st));
      }
      CUDA_TRY(cudaStreamSynchronize(st));
      w.members.clear();
      w.members.push_back(mu);
      w.members.push_back(mg);
      w.glue = HC_GLUE_SILU_MUL;
      w.ws_chunks = -1;
      done[i] = done[j] = 1;
      return HC_OK;
    }

    // ---- plain member
    if (w.glue != HC_GLUE_NONE) { w.members.clear(); w.glue = HC_GLUE_NONE; }
    const bool f8 = d.factor_dtype == HC_FACTORS_FP8;
    for (const Member& o : w.members)
      if (o.slot != d.slot && (o.K != d.K || o.bits != d.bits || o.fp8 != f8))
        return fail(HC_ERR_CONFIG, "mat %d: window members must share K, bits and the factor dtype", i);
    {
      const bool replaces = std::any_of(w.members.begin(), w.members.end(), [&](const Member& o) { return o.slot == d.slot; });
      if (!replaces && (int)w.members.size() >= hc::kMaxMembers)   // checked before the window is touched
        return fail(HC_ERR_CONFIG, "mat %d: window (%d,%d,%d) would have more than %d members", i, d.layer,
                    d.window_kind, d.expert, hc::kMaxMembers);
    }
    Member m = make_member(d);
    const int rows = m.rows();
    CUDA_TRY(m.rec->alloc((size_t)(rows / hc::kRows) * G * hc::rec_bytes(d.bits)));
    if (d.r_stored > 0 && !f8) {
      CUDA_TRY(m.U->alloc((size_t)rows * d.r_stored * 2));
      CUDA_TRY(m.V->alloc((size_t)d.r_stored * d.K * 2));
    }
    Staged sd;
    hc_status s = stage(d, sd, st);
    if (s != HC_OK) return s;
    const int wpr = d.K * d.bits / 32;
    hc::RepackSrc src;
    src.codes[0] = sd.codes + (size_t)d.row_begin * wpr;  src.codes[1] = src.codes[0] + (size_t)8 * wpr;
    src.scales[0] = sd.scales + (size_t)d.row_begin * G;  src.scales[1] = src.scales[0] + (size_t)8 * G;
    src.zeros[0] = sd.zeros + (size_t)d.row_begin * G;    src.zeros[1] = src.zeros[0] + (size_t)8 * G;
    src.U[0] = (sd.U && !f8) ? sd.U + (size_t)d.row_begin * d.r_stored : nullptr;
    src.U[1] = (sd.U && !f8) ? src.U[0] + (size_t)8 * d.r_stored : nullptr;
    src.rstride = hc::kRows;
    CUDA_TRY(hc::launch_repack_records(src, d.K, d.bits, f8 ? 0 : d.r_stored, rows / hc::kRows, (uint8_t*)m.rec->p,
                                       (uint32_t*)m.U->p, st));
    if (f8) {
      const uint8_t* u8 = (const uint8_t*)sd.U + (size_t)d.row_begin * d.r_stored;
      hc_status s8 = load_fp8(m, u8, u8 + (size_t)8 * d.r_stored, hc::kRows, rows / hc::kRows, sd, true, st);
      if (s8 != HC_OK) return s8;
    } else {
      CUDA_TRY(hc::launch_repack_v(sd.V, d.K, d.r_stored, (uint32_t*)m.V->p, st));
    }
    if (d.r_stored > 0 && !f8) {
      CUDA_TRY(m.Vn->alloc((size_t)d.r_stored * d.K * 2));
      CUDA_TRY(hc::launch_repack_vn(sd.V, d.K, d.r_stored, (uint32_t*)m.Vn->p, st));
    }
    // prefill copies are built lazily from the decode records on the first B > 16 call (ensure_prefill)
    CUDA_TRY(cudaStreamSynchronize(st));   // staged temporaries die at scope end
    auto it = std::find_if(w.members.begin(), w.members.end(), [&](const Member& o) { return o.slot == d.slot; });
    if (it != w.members.end()) *it = m; else w.members.push_back(m);
    std::sort(w.members.begin(), w.members.end(), [](const Member& a, const Member& b) { return a.slot < b.slot; });
    w.ws_chunks = -1;
    done[i] = 1;
    return HC_OK;
}

namespace hc {
Options& options() {
  static Options o;
  return o;
}
}  // namespace hc

extern "C" hc_status hc_set_option(const char* name, int32_t value) {
  if (!name) return fail(HC_ERR_CONFIG, "hc_set_option: null name");
  hc::Options& o = hc::options();
  const std::pair<const char*, int*> tab[] = {{"t_forward", &o.t_forward},       {"x_handoff", &o.x_handoff},
                                              {"dep_wait", &o.dep_wait},         {"int8_path", &o.int8_path},
                                              {"prefill_merge", &o.prefill_merge}, {"decode_ctas_per_sm", &o.decode_ctas_per_sm},
                                              {"pdl", &o.pdl}, {"l2_prefetch", &o.l2_prefetch}, {"l2_prefetch_at_start", &o.l2_prefetch_at_start}};
  for (const auto& kv : tab)
    if (std::strcmp(kv.first, name) == 0) {
      if (value < 0) return fail(HC_ERR_CONFIG, "hc_set_option: %s = %d < 0", name, value);
      *kv.second = value;
      ++o.epoch;
      return HC_OK;
    }
  return fail(HC_ERR_CONFIG, "hc_set_option: unknown option '%s'", name);
}

extern "C" hc_status hc_get_option(const char* name, int32_t* value) {
  if (!name || !value) return fail(HC_ERR_CONFIG, "hc_get_option: null argument");
  const hc::Options& o = hc::options();
  const std::pair<const char*, int> tab[] = {{"t_forward", o.t_forward},       {"x_handoff", o.x_handoff},
                                             {"dep_wait", o.dep_wait},         {"int8_path", o.int8_path},
                                             {"prefill_merge", o.prefill_merge}, {"decode_ctas_per_sm", o.decode_ctas_per_sm},
                                             {"pdl", o.pdl}, {"l2_prefetch", o.l2_prefetch}, {"l2_prefetch_at_start", o.l2_prefetch_at_start}};
  for (const auto& kv : tab)
    if (std::strcmp(kv.first, name) == 0) { *value = kv.second; return HC_OK; }
  return fail(HC_ERR_CONFIG, "hc_get_option: unknown option '%s'", name);
}

extern "C" hc_status hc_load_layer(hc_ctx* ctx, const hc_matrix_desc* mats, int32_t n_mats, void* stream) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_load_layer: null context");
  if (n_mats < 0 || (n_mats > 0 && !mats)) return fail(HC_ERR_CONFIG, "hc_load_layer: bad matrix list");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < n_mats; ++i) {
    hc_status s = validate_desc(mats[i], i);
    if (s != HC_OK) return s;
  }
  ctx->invalidate_graphs();
  std::vector<char> done(n_mats, 0);
  for (int i = 0; i < n_mats; ++i) {
    if (done[i]) continue;
    const Key key{mats[i].layer, mats[i].window_kind, mats[i].expert};
    const bool created = ctx->windows.find(key) == ctx->windows.end();
    const hc_status s = load_one(ctx, mats, n_mats, i, done, st);
    if (s != HC_OK) {
      auto it = ctx->windows.find(key);
      if (created && it != ctx->windows.end() && it->second.members.empty()) ctx->windows.erase(it);
      return s;
    }
  }
  return HC_OK;
}

extern "C" hc_status hc_set_rank(hc_ctx* ctx, int32_t layer, int32_t kind, int32_t slot, int32_t expert, int32_t r) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_set_rank: null context");
  auto it = ctx->windows.find(Key{layer, kind, expert});
  if (it == ctx->windows.end()) return fail(HC_ERR_STATE, "hc_set_rank: window (%d,%d,%d) not loaded", layer, kind, expert);
  for (Member& m : it->second.members)
    if (m.slot == slot) {
      if (!admissible_rank(r) || r > m.cap()) return fail(HC_ERR_CONFIG, "hc_set_rank: rank %d not admissible or > cap %d", r, m.cap());
      m.r_alloc = r;
      ctx->invalidate_graphs();
      return HC_OK;
    }
  return fail(HC_ERR_STATE, "hc_set_rank: slot %d not loaded", slot);
}

extern "C" int64_t hc_window_rows(hc_ctx* ctx, int32_t layer, int32_t kind, int32_t expert) {
  if (!ctx) return -1;
  auto it = ctx->windows.find(Key{layer, kind, expert});
  if (it == ctx->windows.end()) return -1;
  return it->second.out_rows();
}

namespace hc {

// t forwarding target: the next window, fed by this window's output columns [lo, hi)
struct FwdSpec {
  Window* next = nullptr;
  int lo = 0, hi = 0;
};

static int window_chunks(const Window& w) {
  int c = 0;
  for (const Member& m : w.members) c += (m.r_alloc + 15) / 16;
  return c;
}

// Whether `next` can receive t from the kernel producing its input (DArgs::fwd / t_in).
static bool forwardable(const Window& next) {
  const int c = window_chunks(next);
  if (c == 0 || c > kFwdMax || (int)next.members.size() > kMaxMembers) return false;
  for (const Member& m : next.members)
    if (m.fp8 || (m.r_alloc > 0 && !(m.Vn && m.Vn->p))) return false;
  return true;
}
static bool can_forward(const Window& next) { return options().t_forward && forwardable(next); }

// Launch arguments of one window (also used by the stack driver).
// x' hand-off between stack windows (DArgs::x16_given / y16)
struct X16Spec {
  const uint16_t* in = nullptr;   // x' of this window written by its producer (or NULL)
  uint16_t* out = nullptr;        // where this window writes the next window's x' (or NULL)
  int lo = 0, hi = 0;             // output columns that are the next window's x
  const unsigned* max_in = nullptr;   // max |x| per (group, batch row) of `in` (DArgs::x16_max), of `out` (y16_max)
  unsigned* max_out = nullptr;
  unsigned* clr = nullptr;            // the max buffer the next window publishes into (zeroed by CTA 0, DArgs::clr_max)
  int clr_n = 0;
};

static hc_status window_args(hc_ctx* ctx, Window& w, const void* x, int ldx, int B, void* y, int y_bf16,
                             const void* resid, int ld_resid, DArgs& a, int& grid, bool t_in = false,
                             const FwdSpec* fw = nullptr, Window* dep = nullptr, bool keep_done = false,
                             const X16Spec* xs16 = nullptr) {
  std::memset(&a, 0, sizeof(a));
  if (xs16) {
    a.x16_given = xs16->in ? 1 : 0;
    a.x16 = xs16->in;
    a.y16 = xs16->out;
    a.y16_lo = xs16->lo;
    a.y16_hi = xs16->hi;
    a.x16_max = xs16->in ? xs16->max_in : nullptr;
    a.y16_max = xs16->out ? xs16->max_out : nullptr;
    a.clr_max = xs16->clr;
    a.clr_n = xs16->clr_n;
  }
  a.t_in = t_in ? 1 : 0;
  a.keep_done = keep_done ? 1 : 0;
  if (dep) {
    if (!dep->cnt.p) return fail(HC_ERR_STATE, "dataflow dependency: producer window workspace missing");
    a.dep_cnt = (unsigned*)dep->cnt.p + 1;
    a.dep_reset = a.dep_cnt;
    int n = 0;
    if (dep->glue == HC_GLUE_SILU_MUL) n = dep->members.front().rows() / 8;
    else for (const Member& m : dep->members) n += m.rows() / kRows;
    a.dep_target = (unsigned)n;
  }
  if (w.members.empty() || (int)w.members.size() > kMaxMembers)
    return fail(HC_ERR_STATE, "window has %d members (1..%d)", (int)w.members.size(), kMaxMembers);
  const Member& m0 = w.members.front();
  a.K = m0.K; a.G = m0.K / kGroup; a.B = B;
  a.x = (const uint16_t*)x; a.ldx = ldx; a.y = y; a.y_bf16 = y_bf16;
  a.resid = (const uint16_t*)resid; a.ld_resid = ld_resid;
  int max_chunks = 0;
  a.n_members = (int)w.members.size();
  if (w.glue == HC_GLUE_SILU_MUL) {
    const Member& up = w.members[0];
    const Member& gate = w.members[1];
    a.glue = 1;
    DMember& d0 = a.m[0];
    d0.rec = (const uint8_t*)up.rec->p; d0.U = (const uint4*)up.U->p; d0.V = (const uint4*)up.V->p;
    d0.n_rb = up.rows() / 8; d0.rb_begin = 0; d0.row_off = 0; d0.r = up.r_alloc; d0.r_stored = up.r_stored;
    d0.chunk_begin = 0;
    d0.us = up.fp8 ? (const float*)up.us->p : nullptr; d0.vs = up.fp8 ? (const float*)up.vs->p : nullptr;
    DMember& d1 = a.m[1];
    d1.rec = nullptr; d1.U = nullptr; d1.V = (const uint4*)gate.V->p;
    d1.n_rb = 0; d1.rb_begin = INT_MAX; d1.row_off = 0; d1.r = gate.r_alloc; d1.r_stored = gate.r_stored;
    d1.chunk_begin = (up.r_alloc + 15) / 16;
    d1.us = gate.fp8 ? (const float*)gate.us->p : nullptr; d1.vs = gate.fp8 ? (const float*)gate.vs->p : nullptr;
    a.fp8 = up.fp8 ? 1 : 0;
    a.n_rb = d0.n_rb;
    a.ldy = up.rows();
    a.n_chunks = d1.chunk_begin + (gate.r_alloc + 15) / 16;
    max_chunks = (up.r_stored + gate.r_stored) / 16;
  } else {
    int rb = 0, row = 0, chunks = 0;
    for (int i = 0; i < a.n_members; ++i) {
      const Member& m = w.members[i];
      DMember& d = a.m[i];
      d.rec = (const uint8_t*)m.rec->p;
      d.U = (const uint4*)m.U->p;
      d.V = (const uint4*)m.V->p;
      d.n_rb = m.rows() / kRows;
      d.rb_begin = rb;
      d.row_off = row;
      d.r = m.r_alloc;
      d.r_stored = m.r_stored;
      d.chunk_begin = chunks;
      d.us = m.fp8 ? (const float*)m.us->p : nullptr;
      d.vs = m.fp8 ? (const float*)m.vs->p : nullptr;
      a.fp8 = m.fp8 ? 1 : 0;
      rb += d.n_rb;
      row += m.rows();
      chunks += (m.r_alloc + 15) / 16;
      max_chunks += m.r_stored / 16;
    }
    a.ldy = row;
    a.n_rb = rb;
    a.n_chunks = chunks;
  }
  if (a.n_chunks > kMaxChunks) return fail(HC_ERR_CONFIG, "window ranks need %d chunks > %d", a.n_chunks, kMaxChunks);
  if (w.ws_chunks < max_chunks) {
    const int mc = std::max(max_chunks, 1);
    CUDA_TRY(w.tacc.alloc(((size_t)hc::kTCopies * mc * hc::kTChunk + 4) * sizeof(long long)));   // [chunk][tier][16][16] + deep flag
    CUDA_TRY(cudaMemset(w.tacc.p, 0, w.tacc.bytes));
    CUDA_TRY(w.cnt.alloc(2 * sizeof(unsigned)));
    CUDA_TRY(cudaMemset(w.cnt.p, 0, w.cnt.bytes));
    w.ws_chunks = max_chunks;
  }
  a.tacc = (long long*)w.tacc.p;
  a.cnt = (unsigned*)w.cnt.p;
  if (!a.x16_given && !decode_stages_x(B, a.K)) {
    const size_t need = (size_t)16 * a.K * 2 + (size_t)16 * a.G * sizeof(float);   // x' [16][K] + 2^σ [G][16]
    if (w.xprep.bytes < need) CUDA_TRY(w.xprep.alloc(need));
    a.x16 = (const uint16_t*)w.xprep.p;
    a.xsig = (float*)((uint16_t*)w.xprep.p + (size_t)16 * a.K);
  }
  if (fw && fw->next) {
    Window& nx = *fw->next;
    const int nch = window_chunks(nx);
    if (nx.ws_chunks < 0 || !nx.tacc.p) return fail(HC_ERR_STATE, "t forwarding: next window workspace missing");
    a.fwd = 1;
    a.fwd_lo = fw->lo;
    a.fwd_hi = fw->hi;
    a.fwd_chunks = nch;
    a.fwd_nm = (int)nx.members.size();
    int cb = 0;
    for (int i = 0; i < a.fwd_nm; ++i) {
      const Member& mm = nx.members[i];
      a.fwd_cb[i] = cb;
      a.fwd_vn[i] = (const uint4*)(mm.Vn ? mm.Vn->p : nullptr);
      a.fwd_rs[i] = mm.r_stored / 16;
      cb += (mm.r_alloc + 15) / 16;
    }
    a.fwd_cb[a.fwd_nm] = cb;
    a.fwd_tacc = (long long*)nx.tacc.p;
  }
  const auto key = std::make_tuple(m0.bits, B, a.K, a.n_chunks, (a.fwd ? a.fwd_chunks : 0) + 1000 * a.x16_given);
  auto it = ctx->max_ctas.find(key);
  if (it == ctx->max_ctas.end())
    it = ctx->max_ctas.emplace(key, decode_max_ctas(m0.bits, B, a.K, a.n_chunks, a.fwd ? a.fwd_chunks : 0,
                                                    a.x16_given != 0)).first;
  if (it->second <= 0) return fail(HC_ERR_RUNTIME, "decode kernel cannot be resident on this device");
  const int n_items = a.n_rb;
  const int per_sm = options().decode_ctas_per_sm;
  const int cap = per_sm > 0 ? std::min(it->second, per_sm * ctx->sms) : it->second;
  grid = std::max(1, std::min(n_items, cap));
  return HC_OK;
}

// L2 prefetch of the next window's records by this launch (DArgs::pf_*; options().l2_prefetch items per CTA).
static void set_prefetch(DArgs& a, const Window* next) {
  const int per_cta = options().l2_prefetch;
  if (!next || per_cta <= 0 || next->members.empty()) return;
  const Member& n0 = next->members.front();
  a.pf_items = per_cta;
  a.pf_at_start = options().l2_prefetch_at_start ? 1 : 0;
  a.pf_item_bytes = (unsigned)((n0.K / kGroup) * rec_bytes(n0.bits));
  if (next->glue == HC_GLUE_SILU_MUL) {   // one record array: 8 up + 8 gate rows per row block
    a.pf_nm = 1;
    a.pf_rec[0] = (const uint8_t*)n0.rec->p;
    a.pf_rb_end[0] = n0.rows() / 8;
    return;
  }
  int cum = 0;
  a.pf_nm = (int)next->members.size();
  for (int i = 0; i < a.pf_nm; ++i) {
    a.pf_rec[i] = (const uint8_t*)next->members[i].rec->p;
    cum += next->members[i].rows() / kRows;
    a.pf_rb_end[i] = cum;
  }
}

static hc_status launch_window(hc_ctx* ctx, Window& w, const void* x, int ldx, int B, void* y, int y_bf16,
                               const void* resid, int ld_resid, cudaStream_t st, bool t_in = false,
                               const FwdSpec* fw = nullptr, Window* dep = nullptr, bool keep_done = false,
                               const X16Spec* xs16 = nullptr, const Window* pf = nullptr) {
  DArgs a;
  int grid = 0;
  hc_status s = window_args(ctx, w, x, ldx, B, y, y_bf16, resid, ld_resid, a, grid, t_in, fw, dep, keep_done, xs16);
  if (s != HC_OK) return s;
  set_prefetch(a, pf);
  a.trace_slot = ctx->trace_slot++;
  if (a.x16 && !a.x16_given)
    CUDA_TRY(launch_xprep(a.x, a.ldx, B, a.K, w.members.front().bits, (uint16_t*)a.x16, a.xsig, st));
  CUDA_TRY(launch_decode(a, w.members.front().bits, grid, st));
  return HC_OK;
}

// Prefill / batched (B > 16) window: per member, T = X·V[:r]ᵀ (tcgen05, fp16 out) then
// Y = X·deq(W)ᵀ + T·U[:, :r]ᵀ (tcgen05, dequant producers + rank slice in the same accumulator).
static hc_status build_prefill_merged(Window& w, cudaStream_t st) {
  PrefillMerged& P = *w.pm;
  std::vector<int> rk;
  for (const Member& m : w.members) rk.push_back(m.r_alloc);
  if (P.valid && P.ranks == rk) return HC_OK;
  const int K = w.members.front().K, G = K / kGroup;
  int N = 0, R = 0;
  for (const Member& m : w.members) { N += m.rows(); R += (m.r_alloc + 15) / 16 * 16; }
  if (R > 256) return fail(HC_ERR_CONFIG, "merged prefill rank slice %d > 256", R);
  CUDA_TRY(P.codes.alloc((size_t)N * (K / 8) * 4));
  CUDA_TRY(P.scales.alloc((size_t)G * N * 2));
  CUDA_TRY(P.zeros.alloc((size_t)G * N));
  if (R > 0) {
    CUDA_TRY(P.V.alloc((size_t)R * K * 2));
    CUDA_TRY(P.U.alloc((size_t)N * R * 2));
    CUDA_TRY(cudaMemsetAsync(P.V.p, 0, P.V.bytes, st));
    CUDA_TRY(cudaMemsetAsync(P.U.p, 0, P.U.bytes, st));
  }
  int row = 0, roff = 0;
  for (const Member& m : w.members) {
    const int rows = m.rows(), r = m.r_alloc;
    CUDA_TRY(cudaMemcpyAsync((uint32_t*)P.codes.p + (size_t)row * (K / 8), m.pcodes->p, (size_t)rows * (K / 8) * 4,
                             cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpy2DAsync((uint16_t*)P.scales.p + row, (size_t)N * 2, m.pscales->p, (size_t)rows * 2, (size_t)rows * 2,
                               G, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaMemcpy2DAsync((uint8_t*)P.zeros.p + row, (size_t)N, m.pzeros->p, (size_t)rows, (size_t)rows, G,
                               cudaMemcpyDeviceToDevice, st));
    if (r > 0) {
      CUDA_TRY(cudaMemcpyAsync((uint16_t*)P.V.p + (size_t)roff * K, m.V16->p, (size_t)r * K * 2, cudaMemcpyDeviceToDevice, st));
      CUDA_TRY(cudaMemcpy2DAsync((uint16_t*)P.U.p + (size_t)row * R + roff, (size_t)R * 2, m.U16->p, (size_t)m.r_stored * 2,
                                 (size_t)r * 2, rows, cudaMemcpyDeviceToDevice, st));
    }
    row += rows;
    roff += (r + 15) / 16 * 16;
  }
  P.R = R;
  P.ranks = rk;
  P.valid = true;
  return HC_OK;
}

static hc_status launch_prefill_window(hc_ctx* ctx, Window& w, const void* x, int M, void* y, int y_dtype,
                                       cudaStream_t st) {
  if (w.glue != HC_GLUE_NONE) return fail(HC_ERR_CONFIG, "prefill of a fused SiLU window is not supported");
  const int K = w.members.front().K;
  for (const Member& m : w.members) {
    if (m.bits != 4) return fail(HC_ERR_CONFIG, "prefill (B > 16) supports 4-bit windows only (got %d-bit)", m.bits);
    if (m.rows() % kPBN) return fail(HC_ERR_CONFIG, "prefill needs member rows %% 256 == 0 (got %d)", m.rows());
  }
  for (Member& m : w.members) {
    hc_status s = ensure_prefill(m, st);
    if (s != HC_OK) return s;
  }
  const size_t xel = (size_t)M * K;
  if (ctx->p_x16.bytes < xel * 2) CUDA_TRY(ctx->p_x16.alloc(xel * 2));
  if (ctx->p_rsig.bytes < (size_t)M * 4) CUDA_TRY(ctx->p_rsig.alloc((size_t)M * 4));
  const float* rsig = (const float*)ctx->p_rsig.p;
  CUDA_TRY(launch_x_rows_f16((const uint16_t*)x, M, K, (uint16_t*)ctx->p_x16.p, (float*)ctx->p_rsig.p, st));
  const int64_t ldy = w.out_rows();
  CUtensorMap tmX, tmV, tmT, tmU;
  if (!encode_tmap_f16(&tmX, ctx->p_x16.p, K, M, K, kPBM)) return fail(HC_ERR_RUNTIME, "tensor map (X) encoding failed");
  int R_merged = 0;
  for (const Member& m : w.members) R_merged += (m.r_alloc + 15) / 16 * 16;
  if (w.members.size() > 1 && R_merged <= 256 && options().prefill_merge) {
    // one GEMM over all members: concatenated rows, stacked rank slices, block-diagonal U
    hc_status s = build_prefill_merged(w, st);
    if (s != HC_OK) return s;
    const PrefillMerged& P = *w.pm;
    const int N = (int)ldy, R = P.R, tw = (R + 63) / 64 * 64;
    CUtensorMap tmC;
    if (!encode_tmap_codes(&tmC, P.codes.p, K / 8, N)) return fail(HC_ERR_RUNTIME, "tensor map (codes) encoding failed");
    if (R > 0) {
      const int tiles_m = (M + kPBM - 1) / kPBM;
      const int ksplit = std::max(1, std::min(K / kPBK / 4, (ctx->sms + tiles_m - 1) / tiles_m));
      if (ctx->p_t16.bytes < (size_t)M * tw * 2) CUDA_TRY(ctx->p_t16.alloc((size_t)M * tw * 2));
      if (ctx->p_tpart.bytes < (size_t)ksplit * M * tw * 4) CUDA_TRY(ctx->p_tpart.alloc((size_t)ksplit * M * tw * 4));
      if (!encode_tmap_f16(&tmV, P.V.p, K, R, K, kPBN)) return fail(HC_ERR_RUNTIME, "tensor map (V) encoding failed");
      PArgs pt{};
      pt.M = M; pt.N = tw; pt.K = K; pt.K2 = 0; pt.n_dim = R; pt.b_mode = 1; pt.ksplit = ksplit;
      pt.out = ctx->p_tpart.p; pt.ldo = tw; pt.out_type = 0;
      pt.tiles_m = tiles_m; pt.tiles_n = 1;
      CUDA_TRY(launch_prefill(tmX, tmV, tmX, tmX, tmC, pt, st));
      CUDA_TRY(launch_splitk_reduce_f16((const float*)ctx->p_tpart.p, ksplit, M, tw, (uint16_t*)ctx->p_t16.p, st));
      if (!encode_tmap_f16(&tmT, ctx->p_t16.p, tw, M, tw, kPBM)) return fail(HC_ERR_RUNTIME, "tensor map (T) encoding failed");
      if (!encode_tmap_f16(&tmU, P.U.p, R, N, R, kPBN)) return fail(HC_ERR_RUNTIME, "tensor map (U) encoding failed");
    }
    PArgs pm{};
    pm.M = M; pm.N = N; pm.K = K; pm.K2 = R; pm.n_dim = kPBN; pm.b_mode = 0; pm.ksplit = 1;
    pm.scales_t = (const uint16_t*)P.scales.p; pm.zeros_t = (const uint8_t*)P.zeros.p;
    pm.out = y; pm.ldo = N; pm.out_type = y_dtype == HC_OUT_F32 ? 0 : 1;
    pm.tiles_m = (M + kPBM - 1) / kPBM; pm.tiles_n = N / kPBN;
    pm.rsig = rsig;
    CUDA_TRY(launch_prefill(tmX, tmX, R > 0 ? tmT : tmX, R > 0 ? tmU : tmX, tmC, pm, st));
    return HC_OK;
  }
  int row_off = 0;
  for (const Member& m : w.members) {
    const int r = m.r_alloc, rpad = (r + 15) / 16 * 16, tw = (rpad + 63) / 64 * 64;
    CUtensorMap tmC;
    if (!encode_tmap_codes(&tmC, m.pcodes->p, K / 8, m.rows())) return fail(HC_ERR_RUNTIME, "tensor map (codes) encoding failed");
    if (r > 0) {
      // T = X·V[:r]ᵀ: one 128 x rpad tile column, split-K over the SMs, deterministic reduce to fp16
      const int tiles_m = (M + kPBM - 1) / kPBM;
      const int ksplit = std::max(1, std::min(K / kPBK / 4, (ctx->sms + tiles_m - 1) / tiles_m));
      if (ctx->p_t16.bytes < (size_t)M * tw * 2) CUDA_TRY(ctx->p_t16.alloc((size_t)M * tw * 2));
      if (ctx->p_tpart.bytes < (size_t)ksplit * M * tw * 4) CUDA_TRY(ctx->p_tpart.alloc((size_t)ksplit * M * tw * 4));
      if (!encode_tmap_f16(&tmV, m.V16->p, K, r, K, kPBN)) return fail(HC_ERR_RUNTIME, "tensor map (V) encoding failed");
      PArgs pt{};
      pt.M = M; pt.N = tw; pt.K = K; pt.K2 = 0; pt.n_dim = rpad; pt.b_mode = 1; pt.ksplit = ksplit;
      pt.out = ctx->p_tpart.p; pt.ldo = tw; pt.out_type = 0;
      pt.tiles_m = tiles_m; pt.tiles_n = 1;
      CUDA_TRY(launch_prefill(tmX, tmV, tmX, tmX, tmC, pt, st));
      CUDA_TRY(launch_splitk_reduce_f16((const float*)ctx->p_tpart.p, ksplit, M, tw, (uint16_t*)ctx->p_t16.p, st));
      if (!encode_tmap_f16(&tmT, ctx->p_t16.p, tw, M, tw, kPBM)) return fail(HC_ERR_RUNTIME, "tensor map (T) encoding failed");
      if (!encode_tmap_f16(&tmU, m.U16->p, r, m.rows(), m.r_stored, kPBN)) return fail(HC_ERR_RUNTIME, "tensor map (U) encoding failed");
    }
    PArgs pm{};
    pm.M = M; pm.N = m.rows(); pm.K = K; pm.K2 = r > 0 ? rpad : 0; pm.n_dim = kPBN; pm.b_mode = 0; pm.ksplit = 1;
    pm.scales_t = (const uint16_t*)m.pscales->p; pm.zeros_t = (const uint8_t*)m.pzeros->p;
    pm.out = y_dtype == HC_OUT_F32 ? (void*)((float*)y + row_off) : (void*)((uint16_t*)y + row_off);
    pm.ldo = (int)ldy; pm.out_type = y_dtype == HC_OUT_F32 ? 0 : 1;
    pm.tiles_m = (M + kPBM - 1) / kPBM; pm.tiles_n = m.rows() / kPBN;
    pm.rsig = rsig;
    CUDA_TRY(launch_prefill(tmX, tmX, r > 0 ? tmT : tmX, r > 0 ? tmU : tmX, tmC, pm, st));
    row_off += m.rows();
  }
  return HC_OK;
}

}  // namespace hc

extern "C" hc_status hc_compensated_linear(hc_ctx* ctx, int32_t layer, int32_t kind, int32_t expert,
                                           const void* x, int32_t B, void* y, int32_t y_dtype, void* stream) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_compensated_linear: null context");
  if (B < 1) return fail(HC_ERR_CONFIG, "hc_compensated_linear: B = %d < 1", B);
  if (y_dtype != HC_OUT_F32 && y_dtype != HC_OUT_BF16) return fail(HC_ERR_CONFIG, "bad y_dtype %d", y_dtype);
  if (!x || !y) return fail(HC_ERR_CONFIG, "hc_compensated_linear: null x or y");
  auto it = ctx->windows.find(Key{layer, kind, expert});
  if (it == ctx->windows.end() || it->second.members.empty())
    return fail(HC_ERR_STATE, "hc_compensated_linear: window (%d,%d,%d) not loaded", layer, kind, expert);
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  Window& w = it->second;
  const int K = w.members.front().K;
  const int64_t rows = w.out_rows();
  const size_t xb = (size_t)B * K * 2, yb = (size_t)B * rows * (y_dtype == HC_OUT_F32 ? 4 : 2);
  const bool hx = !is_device_ptr(x), hy = !is_device_ptr(y);
  const void* dx = x;
  void* dy = y;
  if (hx) {
    if (ctx->stage_x.bytes < xb) CUDA_TRY(ctx->stage_x.alloc(xb));
    CUDA_TRY(cudaMemcpyAsync(ctx->stage_x.p, x, xb, cudaMemcpyHostToDevice, st));
    dx = ctx->stage_x.p;
  }
  if (hy) {
    if (ctx->stage_y.bytes < yb) CUDA_TRY(ctx->stage_y.alloc(yb));
    dy = ctx->stage_y.p;
  }
  hc_status s = B <= 16 ? hc::launch_window(ctx, w, dx, K, B, dy, y_dtype == HC_OUT_BF16, nullptr, 0, st)
                        : hc::launch_prefill_window(ctx, w, dx, B, dy, y_dtype, st);
  if (s != HC_OK) return s;
  if (hy) CUDA_TRY(cudaMemcpyAsync(y, dy, yb, cudaMemcpyDeviceToHost, st));
  if (hx || hy) CUDA_TRY(cudaStreamSynchronize(st));
  return HC_OK;
}

// ------------------------------------------------------------------ grouped MoE
static hc_status moe_tables(hc_ctx* ctx, int layer, hc_ctx::MoECache*& out) {
  hc_ctx::MoECache& c = ctx->moe[layer];
  out = &c;
  if (c.valid) return HC_OK;
  std::vector<hc::MoEExpert> ug, dn;
  int E = 0, cu = 1, cd = 1;
  for (;; ++E) {
    auto fu = ctx->windows.find(Key{layer, HC_WIN_UPGATE, E});
    auto fd = ctx->windows.find(Key{layer, HC_WIN_DOWN, E});
    if (fu == ctx->windows.end() || fd == ctx->windows.end()) break;
    Window& wu = fu->second;
    Window& wd = fd->second;
    if (wu.glue != HC_GLUE_SILU_MUL || wu.members.size() != 2 || wd.members.size() != 1)
      return fail(HC_ERR_STATE, "hc_moe_forward: expert %d of layer %d needs a SiLU-fused UPGATE window and one DOWN matrix", E, layer);
    const Member& up = wu.members[0];
    const Member& gt = wu.members[1];
    const Member& d = wd.members[0];
    if (E == 0) { c.K = up.K; c.F = up.rows(); c.D = d.rows(); c.bits = up.bits; }
    if (up.K != c.K || up.rows() != c.F || d.K != c.F || d.rows() != c.D || up.bits != c.bits || d.bits != c.bits ||
        up.rows() != up.N || d.rows() != d.N)
      return fail(HC_ERR_CONFIG, "hc_moe_forward: experts of layer %d differ in shape / bits (or are sharded)", layer);
    hc::MoEExpert a{}, b{};
    a.rec = (const uint8_t*)up.rec->p; a.U = (const uint4*)up.U->p;
    a.Vn[0] = (const uint4*)(up.Vn ? up.Vn->p : nullptr); a.Vn[1] = (const uint4*)(gt.Vn ? gt.Vn->p : nullptr);
    a.r[0] = up.r_alloc; a.r[1] = gt.r_alloc; a.rs[0] = up.r_stored; a.rs[1] = gt.r_stored;
    b.rec = (const uint8_t*)d.rec->p; b.U = (const uint4*)d.U->p;
    b.Vn[0] = (const uint4*)(d.Vn ? d.Vn->p : nullptr); b.r[0] = d.r_alloc; b.rs[0] = d.r_stored;
    cu = std::max(cu, std::max((up.r_alloc + 15) / 16, (gt.r_alloc + 15) / 16));
    cd = std::max(cd, (d.r_alloc + 15) / 16);
    ug.push_back(a);
    dn.push_back(b);
  }
  if (E == 0) return fail(HC_ERR_STATE, "hc_moe_forward: layer %d has no expert 0 (UPGATE + DOWN windows)", layer);
  if (E > 256) return fail(HC_ERR_CONFIG, "hc_moe_forward: %d experts > 256", E);
  c.E = E;
  c.t_ug = 32 * cu;
  c.t_dn = 32 * cd;
  if (!c.rtilde.empty()) {
    if ((int)c.rtilde.size() != 3 * E)
      return fail(HC_ERR_CONFIG, "hc_moe_forward: dynamic ranks were set for %d experts, layer %d has %d",
                  (int)c.rtilde.size() / 3, layer, E);
    std::vector<int> caps(3 * E);
    for (int e = 0; e < E; ++e) { caps[3 * e] = ug[e].r[0]; caps[3 * e + 1] = ug[e].r[1]; caps[3 * e + 2] = dn[e].r[0]; }
    CUDA_TRY(c.d_rtilde.alloc(c.rtilde.size() * sizeof(float)));
    CUDA_TRY(c.d_caps.alloc(caps.size() * sizeof(int)));
    CUDA_TRY(cudaMemcpy(c.d_rtilde.p, c.rtilde.data(), c.rtilde.size() * sizeof(float), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c.d_caps.p, caps.data(), caps.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  CUDA_TRY(c.ex_ug.alloc(ug.size() * sizeof(hc::MoEExpert)));
  CUDA_TRY(c.ex_dn.alloc(dn.size() * sizeof(hc::MoEExpert)));
  CUDA_TRY(cudaMemcpy(c.ex_ug.p, ug.data(), ug.size() * sizeof(hc::MoEExpert), cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(c.ex_dn.p, dn.data(), dn.size() * sizeof(hc::MoEExpert), cudaMemcpyHostToDevice));
  c.valid = true;
  return HC_OK;
}

extern "C" hc_status hc_moe_set_dynamic_ranks(hc_ctx* ctx, int32_t layer, const float* rtilde, int32_t n_experts,
                                              int32_t k0) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_moe_set_dynamic_ranks: null context");
  hc_ctx::MoECache& c = ctx->moe[layer];
  if (!rtilde) {
    c.rtilde.clear();
    c.valid = false;
    return HC_OK;
  }
  if (n_experts < 1 || n_experts > 256 || k0 < 0 || k0 > 7)
    return fail(HC_ERR_CONFIG, "hc_moe_set_dynamic_ranks: n_experts %d / k0 %d", n_experts, k0);
  for (int i = 0; i < 3 * n_experts; ++i)
    if (!(rtilde[i] >= 0.f) || !(rtilde[i] < 1e30f))
      return fail(HC_ERR_NUMERIC, "hc_moe_set_dynamic_ranks: r̃[%d] = %g is negative or not finite", i, (double)rtilde[i]);
  c.rtilde.assign(rtilde, rtilde + 3 * n_experts);
  c.k0 = k0;
  c.valid = false;                                     // tables (and the device r̃ / caps) rebuilt on next use
  return HC_OK;
}

extern "C" hc_status hc_moe_forward(hc_ctx* ctx, int32_t layer, const void* x, int32_t T, const int32_t* topk_idx,
                                    const float* topk_gate, int32_t topk, void* y, void* stream) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_moe_forward: null context");
  if (T < 1 || T > 1024) return fail(HC_ERR_CONFIG, "hc_moe_forward: T = %d outside [1, 1024]", T);
  if (topk < 1 || topk > hc::kMoEMaxK) return fail(HC_ERR_CONFIG, "hc_moe_forward: topk = %d outside [1, %d]", topk, hc::kMoEMaxK);
  if (!x || !topk_idx || !topk_gate || !y) return fail(HC_ERR_CONFIG, "hc_moe_forward: null pointer");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  hc_ctx::MoECache* c = nullptr;
  hc_status s = moe_tables(ctx, layer, c);
  if (s != HC_OK) return s;
  // entries = Σ_e ceil(n_e / 16) <= min(E, R) + R / 16 (moe_route: chunks of <= 16 rows per expert)
  const int R = T * topk, maxe = std::min(c->E, R) + (R + 15) / 16;
  // workspace carve (256-byte aligned pieces)
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
  const size_t o_nr = take(4), o_ne = take(4), o_rt = take((size_t)R * 4), o_tr = take((size_t)R * 4), o_ee = take((size_t)maxe * 4),
               o_er = take((size_t)maxe * 4), o_ec = take((size_t)maxe * 4), o_xg = take((size_t)R * c->K * 2),
               o_x16 = take((size_t)R * c->K * 2), o_tug = take((size_t)R * c->t_ug * 4), o_m = take((size_t)R * c->F * 2),
               o_md = take((size_t)R * c->F * 2), o_tdn = take((size_t)R * c->t_dn * 4), o_do = take((size_t)R * c->D * 4),
               o_x = take((size_t)T * c->K * 2), o_y = take((size_t)T * c->D * 4), o_rr = take((size_t)R * 3 * sizeof(uint16_t)),
               o_fu = take((size_t)R * (c->K / hc::kGroup) * 4), o_fd = take((size_t)R * (c->F / hc::kGroup) * 4);
  if (ctx->moe_ws.bytes < off) CUDA_TRY(ctx->moe_ws.alloc(off));
  uint8_t* ws = (uint8_t*)ctx->moe_ws.p;
  hc::MoERoute rt;
  rt.n_rows = (int*)(ws + o_nr); rt.n_ent = (int*)(ws + o_ne); rt.row_tok = (int*)(ws + o_rt); rt.tok_row = (int*)(ws + o_tr);
  rt.ent_e = (int*)(ws + o_ee); rt.ent_row0 = (int*)(ws + o_er); rt.ent_ncol = (int*)(ws + o_ec);
  // host inputs are staged (stream-ordered); device inputs are used in place
  const int32_t* didx = topk_idx;
  const float* dgate = topk_gate;
  const void* dx = x;
  void* dy = y;
  const bool hi = !is_device_ptr(topk_idx), hg = !is_device_ptr(topk_gate), hx = !is_device_ptr(x), hy = !is_device_ptr(y);
  if (hi) {
    if (ctx->moe_idx.bytes < (size_t)R * 4) CUDA_TRY(ctx->moe_idx.alloc((size_t)R * 4));
    CUDA_TRY(cudaMemcpyAsync(ctx->moe_idx.p, topk_idx, (size_t)R * 4, cudaMemcpyHostToDevice, st));
    didx = (const int32_t*)ctx->moe_idx.p;
  }
  if (hg) {
    if (ctx->moe_gate.bytes < (size_t)R * 4) CUDA_TRY(ctx->moe_gate.alloc((size_t)R * 4));
    CUDA_TRY(cudaMemcpyAsync(ctx->moe_gate.p, topk_gate, (size_t)R * 4, cudaMemcpyHostToDevice, st));
    dgate = (const float*)ctx->moe_gate.p;
  }
  if (hx) {
    CUDA_TRY(cudaMemcpyAsync(ws + o_x, x, (size_t)T * c->K * 2, cudaMemcpyHostToDevice, st));
    dx = ws + o_x;
  }
  if (hy) dy = ws + o_y;
  const bool dyn = !c->rtilde.empty();
  uint16_t* row_rank = dyn ? (uint16_t*)(ws + o_rr) : nullptr;
  hc::MoEWin wu{(const hc::MoEExpert*)c->ex_ug.p, c->F / 8, c->K, c->K / hc::kGroup, 1, c->t_ug, row_rank, 0};
  hc::MoEWin wd{(const hc::MoEExpert*)c->ex_dn.p, c->D / hc::kRows, c->F, c->F / hc::kGroup, 0, c->t_dn, row_rank, 2};
  hc::MoEDyn mdyn{(const float*)c->d_rtilde.p, (const int*)c->d_caps.p, c->k0, row_rank};
  uint16_t* xg = (uint16_t*)(ws + o_xg);
  uint16_t* x16 = (uint16_t*)(ws + o_x16);
  uint16_t* m = (uint16_t*)(ws + o_m);
  uint16_t* md = (uint16_t*)(ws + o_md);
  float* tug = (float*)(ws + o_tug);
  float* tdn = (float*)(ws + o_tdn);
  float* dout = (float*)(ws + o_do);
  CUDA_TRY(hc::moe_route(didx, dgate, T, topk, c->E, rt, dyn ? &mdyn : nullptr, st));
  ctx->moe_last.T = T; ctx->moe_last.topk = topk; ctx->moe_last.tok_row = rt.tok_row; ctx->moe_last.row_rank = row_rank;
  float* fsu = (float*)(ws + o_fu);
  float* fsd = (float*)(ws + o_fd);
  CUDA_TRY(hc::moe_prep((const uint16_t*)dx, c->K, c->K, c->bits, 1, rt, R, xg, x16, fsu, st));
  CUDA_TRY(hc::moe_rank_proj(wu, rt, maxe, xg, tug, st));
  const int max_cols = std::min(T, 16);                                             // rows of one expert <= T
  CUDA_TRY(hc::moe_gemv(wu, c->bits, rt, maxe, x16, fsu, tug, m, max_cols, st));   // m = bf16(silu(gate)·up)
  CUDA_TRY(hc::moe_prep(m, c->F, c->F, c->bits, 0, rt, R, nullptr, md, fsd, st));
  CUDA_TRY(hc::moe_rank_proj(wd, rt, maxe, m, tdn, st));
  CUDA_TRY(hc::moe_gemv(wd, c->bits, rt, maxe, md, fsd, tdn, dout, max_cols, st)); // DOWN_e(m) per row, fp32
  CUDA_TRY(hc::moe_combine(dout, c->D, dgate, T, topk, rt, (float*)dy, st));
  if (hy) CUDA_TRY(cudaMemcpyAsync(y, dy, (size_t)T * c->D * 4, cudaMemcpyDeviceToHost, st));
  if (hi || hg || hx || hy) CUDA_TRY(cudaStreamSynchronize(st));
  return HC_OK;
}

extern "C" hc_status hc_moe_last_ranks(hc_ctx* ctx, int32_t* out, int32_t T, int32_t topk) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_moe_last_ranks: null context");
  if (!out) return fail(HC_ERR_CONFIG, "hc_moe_last_ranks: null output");
  const auto& L = ctx->moe_last;
  if (!L.row_rank) return fail(HC_ERR_STATE, "hc_moe_last_ranks: the last hc_moe_forward ran without dynamic ranks");
  if (T != L.T || topk != L.topk) return fail(HC_ERR_CONFIG, "hc_moe_last_ranks: T/topk %d/%d != last call's %d/%d", T, topk, L.T, L.topk);
  CUDA_TRY(cudaSetDevice(ctx->device));
  CUDA_TRY(cudaDeviceSynchronize());
  const int R = T * topk;
  std::vector<int> tok_row(R);
  std::vector<uint16_t> rr((size_t)R * 3);
  CUDA_TRY(cudaMemcpy(tok_row.data(), L.tok_row, (size_t)R * sizeof(int), cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(rr.data(), L.row_rank, rr.size() * sizeof(uint16_t), cudaMemcpyDeviceToHost));
  for (int i = 0; i < R; ++i)
    for (int sl = 0; sl < 3; ++sl) out[(size_t)i * 3 + sl] = tok_row[i] < 0 ? -1 : (int32_t)rr[(size_t)tok_row[i] * 3 + sl];
  return HC_OK;
}

// ------------------------------------------------------------------ decode stack
namespace {

struct LayerPlan {
  Window *qkv, *o, *ug, *down;
};

hc_status stack_plan(hc_ctx* ctx, std::vector<LayerPlan>& plan, int& d, int& nqkv, int& f, bool check_shard = true) {
  plan.clear();
  for (int l = 0;; ++l) {
    auto f0 = ctx->windows.find(Key{l, HC_WIN_QKV, -1});
    if (f0 == ctx->windows.end()) break;
    auto f1 = ctx->windows.find(Key{l, HC_WIN_O, -1});
    auto f2 = ctx->windows.find(Key{l, HC_WIN_UPGATE, -1});
    auto f3 = ctx->windows.find(Key{l, HC_WIN_DOWN, -1});
    if (f1 == ctx->windows.end() || f2 == ctx->windows.end() || f3 == ctx->windows.end())
      return fail(HC_ERR_STATE, "hc_stack_forward: layer %d lacks a window", l);
    if (f2->second.glue != HC_GLUE_SILU_MUL)
      return fail(HC_ERR_STATE, "hc_stack_forward: layer %d UPGATE window is not loaded with HC_GLUE_SILU_MUL", l);
    plan.push_back(LayerPlan{&f0->second, &f1->second, &f2->second, &f3->second});
  }
  if (plan.empty()) return fail(HC_ERR_STATE, "hc_stack_forward: no layer 0 QKV window loaded");
  // full (unsharded) widths: G x the local rows of every member
  const int G = ctx->world;
  const LayerPlan& p0 = plan.front();
  d = p0.qkv->members.front().K;
  nqkv = (int)(G * p0.qkv->out_rows());
  f = (int)(G * p0.ug->out_rows());
  for (size_t l = 0; l < plan.size(); ++l) {
    const LayerPlan& p = plan[l];
    const int q_rows = G * p.qkv->members.front().rows();
    if (p.qkv->members.front().K != d || G * p.qkv->out_rows() != nqkv || q_rows != d || p.o->members.front().K != d ||
        G * p.o->out_rows() != d || p.ug->members.front().K != d || G * p.ug->out_rows() != f ||
        p.down->members.front().K != f || G * p.down->out_rows() != d)
      return fail(HC_ERR_CONFIG, "hc_stack_forward: layer %zu shapes inconsistent (need q rows = hidden = O/DOWN rows)", l);
    if (G > 1 && check_shard)
      for (Window* w : {p.qkv, p.o, p.ug, p.down})
        for (const Member& m : w->members)
          if (G * m.rows() != m.N || m.row_begin != ctx->rank * m.rows())
            return fail(HC_ERR_CONFIG, "hc_stack_forward: layer %zu member not column-sharded as rows [rank*N/G, (rank+1)*N/G)", l);
  }
  return HC_OK;
}

// ---- peer mode: gather fused into the decode epilogue over peer memory
static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

// Region layout for the loaded stack sharded over G ranks (identical on every rank).
static hc_status peer_layout(hc_ctx* ctx, int G, hc_ctx::Peer& P) {
  const int saved_w = ctx->world;
  ctx->world = G;
  std::vector<LayerPlan> plan;
  int d = 0, nqkv = 0, f = 0;
  hc_status s = stack_plan(ctx, plan, d, nqkv, f, false);   // the rank is checked by hc_peer_set / connect
  ctx->world = saved_w;
  if (s != HC_OK) return s;
  int mc = 1;
  for (const LayerPlan& p : plan)
    for (Window* w : {p.qkv, p.o, p.ug, p.down}) {
      int c = 0;
      for (const Member& m : w->members) c += m.r_stored / 16;
      mc = std::max(mc, c);
    }
  size_t off = 0;
  P.off_qkv = off; off += align256((size_t)16 * nqkv * 2);
  P.off_h1 = off;  off += align256((size_t)16 * d * 2);
  P.off_m = off;   off += align256((size_t)16 * f * 2);
  P.off_h = off;   off += align256((size_t)16 * d * 2);
  P.off_win = off;
  P.win_stride = align256(128 + ((size_t)hc::kTCopies * mc * hc::kTChunk + 4) * sizeof(long long));
  P.n_win = 4 * (int)plan.size();
  P.mc = mc;
  P.G = G;
  P.bytes = off + (size_t)P.n_win * P.win_stride;
  return HC_OK;
}
static unsigned* peer_cnt(const hc_ctx::Peer& P, int q, int wi) {
  return (unsigned*)((uint8_t*)P.base[q] + P.off_win + (size_t)wi * P.win_stride);
}
static long long* peer_tacc(const hc_ctx::Peer& P, int q, int wi) {
  return (long long*)((uint8_t*)P.base[q] + P.off_win + (size_t)wi * P.win_stride + 128);
}
static uint16_t* peer_act(const hc_ctx::Peer& P, int q, size_t off) { return (uint16_t*)((uint8_t*)P.base[q] + off); }

// Rows of the gather one rank contributes for window w (the consumer waits for G times this).
static unsigned local_row_blocks(const Window& w) {
  if (w.glue == HC_GLUE_SILU_MUL) return (unsigned)(w.members.front().rows() / 8);
  unsigned n = 0;
  for (const Member& m : w.members) n += (unsigned)(m.rows() / hc::kRows);
  return n;
}

// One peer-mode window: local rows, outputs to every rank's gathered buffer (act_off), t partials of this
// rank's slice to every rank's next-window accumulators, and the gather counters.
static hc_status peer_window(hc_ctx* ctx, Window& w, int wi, const void* x, int ldx, int B, size_t act_off, int ld_full,
                             const void* resid, int ld_resid, const Window* dep, bool t_in, Window* next, int fwd_lo,
                             int fwd_hi, cudaStream_t st) {
  const hc_ctx::Peer& P = ctx->peer;
  const int G = P.G, rank = ctx->rank;
  const bool fwd = next && hc::forwardable(*next);
  hc::FwdSpec fs{fwd ? next : nullptr, fwd_lo, fwd_hi};
  hc::DArgs a;
  int grid = 0;
  hc_status s = hc::window_args(ctx, w, x, ldx, B, peer_act(P, rank, act_off), 1, resid, ld_resid, a, grid, t_in,
                            fwd ? &fs : nullptr);
  if (s != HC_OK) return s;
  hc::set_prefetch(a, next);
  if (a.n_chunks > P.mc || (fwd && a.fwd_chunks > P.mc))
    return fail(HC_ERR_STATE, "peer mode: ranks exceed the peer region's t accumulators (call hc_peer_region again)");
  a.npeer = G;
  a.ld_full = ld_full;
  for (int q = 0; q < G; ++q) {
    a.ypeer[q] = peer_act(P, q, act_off);
    a.dpeer[q] = peer_cnt(P, q, wi);
    if (fwd) a.fwdpeer[q] = peer_tacc(P, q, wi + 1);
  }
  a.tacc = peer_tacc(P, rank, wi);
  if (fwd) a.fwd_tacc = peer_tacc(P, rank, wi + 1);
  // output columns in the full gathered window output: member m's local rows start at F(m) + rank·rows(m)
  if (a.glue) {
    a.m[0].full_off = rank * (int)w.out_rows();
  } else {
    int F = 0;
    for (int i = 0; i < a.n_members; ++i) {
      a.m[i].full_off = F + rank * w.members[i].rows();
      F += G * w.members[i].rows();
    }
  }
  unsigned* dep_cnt = dep ? peer_cnt(P, rank, wi - 1) : nullptr;
  const unsigned target = dep ? (unsigned)G * local_row_blocks(*dep) : 0u;
  a.dep_reset = dep_cnt;
  a.trace_slot = ctx->trace_slot++;
  if (a.x16 && !a.x16_given) {
    // unstaged x: the x-prep kernel waits for the gather; the decode launch follows it in stream order
    a.dep_cnt = nullptr;
    CUDA_TRY(hc::launch_xprep(a.x, a.ldx, B, a.K, w.members.front().bits, (uint16_t*)a.x16, a.xsig, st, dep_cnt, target));
  } else {
    a.dep_cnt = dep_cnt;
    a.dep_target = target;
  }
  CUDA_TRY(hc::launch_decode(a, w.members.front().bits, grid, st));
  return HC_OK;
}

// One window of a column-sharded stack: local rows -> NCCL all-gather -> canonical full layout.
static hc_status tp_window(hc_ctx* ctx, Window& w, const void* x, int ldx, int B, void* full_out, const void* resid_full,
                           int ld_resid, cudaStream_t st) {
  const int n_local = (int)w.out_rows();
  uint16_t* send = (uint16_t*)ctx->t_send.p;
  const void* resid = resid_full ? (const void*)((const uint16_t*)resid_full + (size_t)ctx->rank * n_local) : nullptr;
  hc_status s = hc::launch_window(ctx, w, x, ldx, B, send, 1, resid, ld_resid, st);
  if (s != HC_OK) return s;
  char msg[256];
  if (!hc::comm_allgather_bf16(ctx->comm, send, ctx->t_gather.p, (size_t)B * n_local, st, msg, sizeof(msg)))
    return fail(HC_ERR_RUNTIME, "%s", msg);
  hc::GatherPlan gp{};
  gp.G = ctx->world; gp.B = B; gp.n_local = n_local;
  if (w.glue == HC_GLUE_SILU_MUL) {
    gp.n_members = 1; gp.w[0] = n_local; gp.o[0] = 0;
  } else {
    gp.n_members = (int)w.members.size();
    int o = 0;
    for (int i = 0; i < gp.n_members; ++i) { gp.w[i] = w.members[i].rows(); gp.o[i] = o; o += gp.w[i]; }
  }
  CUDA_TRY(hc::launch_unshard((const uint16_t*)ctx->t_gather.p, (uint16_t*)full_out, gp, st));
  return HC_OK;
}

}  // namespace

// dev-only (not in hcinfer.h): point the stack kernel's trace stamps at a device buffer
extern "C" int hc_dev_decode_trace(void* buf) { return (int)hc::decode_set_trace(buf); }

extern "C" hc_status hc_stack_forward(hc_ctx* ctx, const void* x, int32_t B, void* y, void* stream) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_stack_forward: null context");
  if (B < 1 || B > 16) return fail(HC_ERR_CONFIG, "hc_stack_forward: B = %d outside [1, 16]", B);
  if (!x || !y) return fail(HC_ERR_CONFIG, "hc_stack_forward: null x or y");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<LayerPlan> plan;
  int d = 0, nqkv = 0, f = 0;
  hc_status s = stack_plan(ctx, plan, d, nqkv, f);
  if (s != HC_OK) return s;
  const size_t hb = (size_t)B * d * 2;
  const bool hx = !is_device_ptr(x), hy = !is_device_ptr(y);
  const void* dx = x;
  void* dy = y;
  if (hx) {
    if (ctx->stage_x.bytes < hb) CUDA_TRY(ctx->stage_x.alloc(hb));
    CUDA_TRY(cudaMemcpyAsync(ctx->stage_x.p, x, hb, cudaMemcpyHostToDevice, st));
    dx = ctx->stage_x.p;
  }
  if (hy) {
    if (ctx->stage_y.bytes < hb) CUDA_TRY(ctx->stage_y.alloc(hb));
    dy = ctx->stage_y.p;
  }
  if (ctx->s_h.bytes < (size_t)16 * d * 2) {
    ctx->invalidate_graphs();
    CUDA_TRY(ctx->s_h.alloc((size_t)16 * d * 2));
    CUDA_TRY(ctx->s_h1.alloc((size_t)16 * d * 2));
  }
  if (ctx->s_qkv.bytes < (size_t)16 * nqkv * 2) { ctx->invalidate_graphs(); CUDA_TRY(ctx->s_qkv.alloc((size_t)16 * nqkv * 2)); }
  if (ctx->s_m.bytes < (size_t)16 * f * 2) { ctx->invalidate_graphs(); CUDA_TRY(ctx->s_m.alloc((size_t)16 * f * 2)); }
  {
    const size_t xb[4] = {(size_t)16 * d * 2, (size_t)16 * d * 2, (size_t)16 * f * 2, (size_t)16 * d * 2};
    for (int i = 0; i < 4; ++i)
      if (ctx->s_x16[i].bytes < xb[i]) { ctx->invalidate_graphs(); CUDA_TRY(ctx->s_x16[i].alloc(xb[i])); }
    const size_t mb = (size_t)4 * (std::max(d, f) / hc::kGroup) * 16 * sizeof(unsigned);
    if (ctx->s_x16max.bytes < mb) {
      ctx->invalidate_graphs();
      CUDA_TRY(ctx->s_x16max.alloc(mb));
      CUDA_TRY(cudaMemset(ctx->s_x16max.p, 0, mb));
    }
  }
  const bool tp = ctx->comm != nullptr && !ctx->peer.on;
  if (tp) {
    const size_t widest = (size_t)std::max(std::max(nqkv, f), d);   // full width of any window output
    if (ctx->t_send.bytes < (size_t)16 * widest * 2) { ctx->invalidate_graphs(); CUDA_TRY(ctx->t_send.alloc((size_t)16 * widest * 2)); }
    if (ctx->t_gather.bytes < (size_t)16 * widest * 2) { ctx->invalidate_graphs(); CUDA_TRY(ctx->t_gather.alloc((size_t)16 * widest * 2)); }
  }

  auto key = std::make_tuple((int)B, dx, dy);
  auto git = ctx->graphs.find(key);
  if (git != ctx->graphs.end() && git->second->epoch != hc::options().epoch) {   // options changed: re-plan
    ctx->graphs.erase(git);
    git = ctx->graphs.end();
  }
  if (git == ctx->graphs.end()) {
    // first use: make sure every window's workspace exists (allocation is not capturable), then
    // capture the 4·L launches into one graph
    for (LayerPlan& p : plan)
      for (Window* w : {p.qkv, p.o, p.ug, p.down}) {
        hc::DArgs a;
        int grid;
        s = hc::window_args(ctx, *w, dx, d, B, dy, 1, nullptr, 0, a, grid);
        if (s != HC_OK) return s;
      }
    cudaStream_t cs = ctx->cap_stream;
    CUDA_TRY(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    hc_status cap = HC_OK;
    const uint16_t* hin = (const uint16_t*)dx;
    uint16_t* h = (uint16_t*)ctx->s_h.p;
    uint16_t* h1 = (uint16_t*)ctx->s_h1.p;
    uint16_t* qkv = (uint16_t*)ctx->s_qkv.p;
    uint16_t* mm = (uint16_t*)ctx->s_m.p;
    for (size_t l = 0; l < plan.size() && cap == HC_OK; ++l) {
      LayerPlan& p = plan[l];
      uint16_t* hout = (l + 1 == plan.size()) ? (uint16_t*)dy : h;
      if (ctx->peer.on) {
        // peer mode: every window gathers through peer memory; t of the next window is exchanged as partials
        const hc_ctx::Peer& P = ctx->peer;
        const int rk = ctx->rank;
        const int wi = 4 * (int)l;
        uint16_t* aq = peer_act(P, rk, P.off_qkv), *ah1 = peer_act(P, rk, P.off_h1), *am = peer_act(P, rk, P.off_m),
                  *ah = peer_act(P, rk, P.off_h);
        const uint16_t* hx_in = l == 0 ? (const uint16_t*)dx : ah;
        Window* nq = l + 1 < plan.size() ? plan[l + 1].qkv : nullptr;
        const bool tq = l > 0 && hc::forwardable(*p.qkv);
        cap = peer_window(ctx, *p.qkv, wi, hx_in, d, B, P.off_qkv, nqkv, nullptr, 0, l > 0 ? plan[l - 1].down : nullptr,
                          tq, p.o, 0, d, cs);                                                        // q | k | v
        if (cap == HC_OK)
          cap = peer_window(ctx, *p.o, wi + 1, aq, nqkv, B, P.off_h1, d, hx_in, d, p.qkv, hc::forwardable(*p.o), p.ug, 0, d,
                            cs);                                                                     // h1 = h + O(q)
        if (cap == HC_OK)
          cap = peer_window(ctx, *p.ug, wi + 2, ah1, d, B, P.off_m, f, nullptr, 0, p.o, hc::forwardable(*p.ug), p.down, 0, f,
                            cs);                                                                     // m = silu(g)·u
        if (cap == HC_OK)
          cap = peer_window(ctx, *p.down, wi + 3, am, f, B, P.off_h, d, ah1, d, p.ug, hc::forwardable(*p.down), nq, 0, d,
                            cs);                                                                     // h' = h1 + DOWN(m)
        if (cap == HC_OK && l + 1 == plan.size()) {
          const cudaError_t e0 = hc::launch_peer_wait_copy(peer_cnt(P, rk, wi + 3), (unsigned)P.G * local_row_blocks(*p.down),
                                                           peer_cnt(P, rk, wi + 3), ah, (uint16_t*)dy, (size_t)B * d, cs);
          if (e0 != cudaSuccess) cap = fail(HC_ERR_RUNTIME, "peer gather wait: %s", cudaGetErrorString(e0));
        }
      } else if (!tp) {
        // t forwarding: each window's epilogue accumulates the next window's t = V·x from
        // the outputs it writes, so only layer 0's QKV computes its own V·x
        const bool f_o = hc::can_forward(*p.o), f_ug = hc::can_forward(*p.ug), f_dn = hc::can_forward(*p.down);
        const bool f_q = l + 1 < plan.size() && hc::can_forward(*plan[l + 1].qkv);
        const bool t_q = l > 0 && hc::can_forward(*p.qkv);
        const hc::FwdSpec s_o{f_o ? p.o : nullptr, 0, d}, s_ug{f_ug ? p.ug : nullptr, 0, d},
            s_dn{f_dn ? p.down : nullptr, 0, f}, s_q{f_q ? plan[l + 1].qkv : nullptr, 0, d};
        // dataflow dependencies: a window whose x is staged in shared memory waits on
        // its producer's row-block counter instead of the kernel boundary (an unstaged window keeps the
        // grid dependency: its x-prep kernel sits in between)
        const bool dx_ok = hc::options().dep_wait != 0;
        const bool hx_ok = dx_ok && hc::options().x_handoff != 0;
        const bool sx_q = dx_ok && hc::decode_stages_x(B, d), sx_f = dx_ok && hc::decode_stages_x(B, f);
        Window* prev_dn = l > 0 ? plan[l - 1].down : nullptr;
        const bool next_q = l + 1 < plan.size() && sx_q;
        ctx->trace_slot = (int)(4 * l);
        // x' hand-off: every window but layer 0's QKV reads the fp16 x' its producer's
        // epilogue wrote (no staging, no x-prep kernel); it then waits for the producer's counter itself
        const bool hx = hx_ok;
        uint16_t* xq16 = (uint16_t*)ctx->s_x16[0].p, *xh1 = (uint16_t*)ctx->s_x16[1].p;
        uint16_t* xm16 = (uint16_t*)ctx->s_x16[2].p, *xh16 = (uint16_t*)ctx->s_x16[3].p;
        // int8-path windows (decode_uses_i8) stage bf16 x themselves: no x' hand-off into them
        auto i8w = [&](Window* w) { return hc::decode_uses_i8(w->members.front().bits, B, w->members.front().K); };
        const bool i8q = i8w(p.qkv), i8o = i8w(p.o), i8ug = i8w(p.ug), i8dn = i8w(p.down);
        const bool i8qn = l + 1 < plan.size() ? i8w(plan[l + 1].qkv) : true;
        // x' range (R20): max |x| per (group, batch row) of q, h1, m, h; window w zeroes the buffer window w+1
        // publishes into (layer 0's QKV output buffer is zeroed by a memset at the start of the graph)
        const int gm = std::max(d, f) / hc::kGroup;
        unsigned* xmx = (unsigned*)ctx->s_x16max.p;
        unsigned* mq = xmx, *mh1 = xmx + (size_t)gm * 16, *mm16 = xmx + (size_t)2 * gm * 16, *mh = xmx + (size_t)3 * gm * 16;
        if (l == 0) {
          const cudaError_t e0 = cudaMemsetAsync(mq, 0, (size_t)gm * 16 * sizeof(unsigned), cs);
          if (e0 != cudaSuccess) { cap = fail(HC_ERR_RUNTIME, "x' max reset: %s", cudaGetErrorString(e0)); break; }
        }
        const int nd = d / hc::kGroup * 16, nf = f / hc::kGroup * 16;
        const hc::X16Spec x_q{hx && l > 0 && !i8q ? xh16 : nullptr, hx && !i8o ? xq16 : nullptr, 0, d, mh, mq, mh1, nd};
        const hc::X16Spec x_o{hx && !i8o ? xq16 : nullptr, hx && !i8ug ? xh1 : nullptr, 0, d, mq, mh1, mm16, nf};
        const hc::X16Spec x_ug{hx && !i8ug ? xh1 : nullptr, hx && !i8dn ? xm16 : nullptr, 0, f, mh1, mm16, mh, nd};
        const hc::X16Spec x_dn{hx && !i8dn ? xm16 : nullptr, (hx && !i8qn) ? xh16 : nullptr, 0, d, mm16, mh,
                               l + 1 < plan.size() ? mq : nullptr, nd};
        const bool dq = sx_q || (hx && l > 0), do_ = sx_q || hx, dug = sx_q || hx, ddn = sx_f || hx;
        const bool kq = sx_q || hx, ko = sx_q || hx, kug = sx_f || hx;     // keep(producer) = dep(consumer)
        const bool kdn = l + 1 < plan.size() && (sx_q || hx);
        const Window* nqw = l + 1 < plan.size() ? plan[l + 1].qkv : nullptr;
        cap = hc::launch_window(ctx, *p.qkv, hin, d, B, qkv, 1, nullptr, 0, cs, t_q, &s_o,
                                (prev_dn && dq) ? prev_dn : nullptr, kq, &x_q, p.o);                   // q | k | v
        if (cap == HC_OK) cap = hc::launch_window(ctx, *p.o, qkv, nqkv, B, h1, 1, hin, d, cs, f_o, &s_ug,
                                                  do_ ? p.qkv : nullptr, ko, &x_o, p.ug);              // h1 = h + O(q)
        if (cap == HC_OK) cap = hc::launch_window(ctx, *p.ug, h1, d, B, mm, 1, nullptr, 0, cs, f_ug, &s_dn,
                                                  dug ? p.o : nullptr, kug, &x_ug, p.down);            // m = silu(g)·u
        if (cap == HC_OK) cap = hc::launch_window(ctx, *p.down, mm, f, B, hout, 1, h1, d, cs, f_dn, &s_q,
                                                  ddn ? p.ug : nullptr, kdn, &x_dn, nqw);              // h' = h1 + DOWN(m)
      } else {                                                   // column-sharded: gather every window
        cap = tp_window(ctx, *p.qkv, hin, d, B, qkv, nullptr, 0, cs);
        if (cap == HC_OK) cap = tp_window(ctx, *p.o, qkv, nqkv, B, h1, hin, d, cs);
        if (cap == HC_OK) cap = tp_window(ctx, *p.ug, h1, d, B, mm, nullptr, 0, cs);
        if (cap == HC_OK) cap = tp_window(ctx, *p.down, mm, f, B, hout, h1, d, cs);
      }
      hin = hout;
    }
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g);
    if (cap != HC_OK) { if (g) cudaGraphDestroy(g); return cap; }
    CUDA_TRY(e);
    std::unique_ptr<StackGraph> sg(new StackGraph());
    sg->epoch = hc::options().epoch;
    e = cudaGraphInstantiate(&sg->exec, g, 0);
    cudaGraphDestroy(g);
    CUDA_TRY(e);
    git = ctx->graphs.emplace(key, std::move(sg)).first;
  }
  CUDA_TRY(cudaGraphLaunch(git->second->exec, st));
  if (hy) CUDA_TRY(cudaMemcpyAsync(y, dy, hb, cudaMemcpyDeviceToHost, st));
  if (hx || hy) CUDA_TRY(cudaStreamSynchronize(st));
  return HC_OK;
}

// ------------------------------------------------------------------ calibration
extern "C" hc_status hc_calib_svd(hc_ctx* ctx, const float* W, const uint32_t* codes, const uint16_t* scales,
                                  const uint8_t* zeros, int32_t n_mats, int32_t N, int32_t K, int32_t bits,
                                  int32_t group, int32_t r, double* U_out, double* V_out, double* sigma_out,
                                  int32_t* sweeps_out, void* stream) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_calib_svd: null context");
  if (n_mats < 1 || N < 32 || K < 32 || N % 32 || K % 32)
    return fail(HC_ERR_CONFIG, "hc_calib_svd: n_mats %d, N %d, K %d (N, K multiples of 32)", n_mats, N, K);
  if (!(bits == 2 || bits == 3 || bits == 4 || bits == 8) || group < 1 || K % group || (K * bits) % 32)
    return fail(HC_ERR_CONFIG, "hc_calib_svd: bits %d / group %d", bits, group);
  if (r < 0 || r > std::min(N, K)) return fail(HC_ERR_CONFIG, "hc_calib_svd: rank %d outside [0, min(N, K)]", r);
  if (!W || !codes || !scales || !zeros || (r > 0 && (!U_out || !V_out)))
    return fail(HC_ERR_CONFIG, "hc_calib_svd: null input / output");
  for (const void* p : {(const void*)W, (const void*)codes, (const void*)scales, (const void*)zeros})
    if (!is_device_ptr(p)) return fail(HC_ERR_CONFIG, "hc_calib_svd: inputs must be device pointers");
  CUDA_TRY(cudaSetDevice(ctx->device));
  const size_t need = hc::calib_workspace_bytes(n_mats, N, K, r);
  if (ctx->calib_ws.bytes < need) CUDA_TRY(ctx->calib_ws.alloc(need));
  hc::CalibSvdArgs a{W, codes, scales, zeros, n_mats, N, K, bits, group, r, U_out, V_out, sigma_out, 40, 1e-15};
  int sweeps = 0;
  CUDA_TRY(hc::calib_svd(a, ctx->calib_ws.p, (cudaStream_t)stream, &sweeps));
  if (sweeps_out) *sweeps_out = sweeps;
  return HC_OK;
}

extern "C" hc_status hc_calib_salience(hc_ctx* ctx, const double* sigma, int32_t n_mats, int32_t n, double tau,
                                       double* phi_out, int32_t* n_salient_out, void* stream) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_calib_salience: null context");
  if (n_mats < 1 || n < 1 || !sigma || !phi_out || !n_salient_out || !std::isfinite(tau))
    return fail(HC_ERR_CONFIG, "hc_calib_salience: bad arguments");
  CUDA_TRY(cudaSetDevice(ctx->device));
  CUDA_TRY(hc::calib_salience(sigma, n_mats, n, tau, phi_out, n_salient_out, (cudaStream_t)stream));
  return HC_OK;
}

extern "C" hc_status hc_calib_r_std(const int32_t* Ns, int32_t n_members, int32_t K, int32_t bits, int32_t group,
                                    double eps, double* r_std_out) {
  if (!Ns || n_members < 1 || !r_std_out || K < 1 || group < 1 || K % group || !(eps > 0.0) || !std::isfinite(eps))
    return fail(HC_ERR_CONFIG, "hc_calib_r_std: bad arguments");
  if (!(bits == 2 || bits == 3 || bits == 4 || bits == 8)) return fail(HC_ERR_CONFIG, "hc_calib_r_std: bits %d", bits);
  long long bytes = 0, nsum = 0;
  for (int i = 0; i < n_members; ++i) {
    if (Ns[i] < 1) return fail(HC_ERR_CONFIG, "hc_calib_r_std: N[%d] = %d", i, Ns[i]);
    const long long N = Ns[i];
    bytes += N * K * bits / 8 + N * (K / group) * (16 + bits) / 8;
    nsum += N;
  }
  const double nbar = (double)nsum / (double)n_members;
  *r_std_out = std::floor(eps * (double)bytes / (2.0 * (nbar + (double)K)));
  return HC_OK;
}

// ------------------------------------------------------------------ peer mode
extern "C" hc_status hc_peer_region(hc_ctx* ctx, int32_t world, void** base_out, uint64_t* bytes_out) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_peer_region: null context");
  if (world < 2 || world > hc::kMaxPeers) return fail(HC_ERR_CONFIG, "hc_peer_region: world %d outside [2, %d]", world, hc::kMaxPeers);
  CUDA_TRY(cudaSetDevice(ctx->device));
  hc_ctx::Peer& P = ctx->peer;
  for (void* p : P.opened) cudaIpcCloseMemHandle(p);
  P.opened.clear();
  P.on = false;
  hc_status s = peer_layout(ctx, world, P);
  if (s != HC_OK) return s;
  CUDA_TRY(P.region.alloc(P.bytes));
  CUDA_TRY(cudaMemset(P.region.p, 0, P.bytes));
  ctx->invalidate_graphs();
  if (base_out) *base_out = ctx->peer.region.p;
  if (bytes_out) *bytes_out = (uint64_t)ctx->peer.bytes;
  return HC_OK;
}

static hc_status peer_enable(hc_ctx* ctx, int32_t rank, int32_t world) {
  ctx->rank = rank;
  ctx->world = world;
  ctx->peer.on = true;
  ctx->invalidate_graphs();
  std::vector<LayerPlan> plan;
  int d = 0, nqkv = 0, f = 0;
  hc_status s = stack_plan(ctx, plan, d, nqkv, f);   // the loaded rows must be this rank's shard
  if (s != HC_OK) { ctx->peer.on = false; ctx->world = 1; ctx->rank = 0; }
  return s;
}

extern "C" hc_status hc_peer_set(hc_ctx* ctx, int32_t rank, int32_t world, void* const* bases) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_peer_set: null context");
  if (!ctx->peer.region.p || ctx->peer.G != world) return fail(HC_ERR_STATE, "hc_peer_set: call hc_peer_region(world) first");
  if (rank < 0 || rank >= world || !bases) return fail(HC_ERR_CONFIG, "hc_peer_set: rank %d / world %d", rank, world);
  if (bases[rank] != ctx->peer.region.p) return fail(HC_ERR_CONFIG, "hc_peer_set: bases[rank] is not this context's region");
  for (int q = 0; q < world; ++q) {
    if (!bases[q]) return fail(HC_ERR_CONFIG, "hc_peer_set: null base of rank %d", q);
    ctx->peer.base[q] = bases[q];
  }
  return peer_enable(ctx, rank, world);
}

extern "C" hc_status hc_peer_ipc_handle(hc_ctx* ctx, uint8_t* out64) {
  if (!ctx || !out64) return fail(HC_ERR_CONFIG, "hc_peer_ipc_handle: null argument");
  if (!ctx->peer.region.p) return fail(HC_ERR_STATE, "hc_peer_ipc_handle: no peer region");
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, ctx->peer.region.p));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(out64, &h, 64);
  return HC_OK;
}

extern "C" hc_status hc_peer_connect(hc_ctx* ctx, int32_t rank, int32_t world, const uint8_t* handles) {
  if (!ctx || !handles) return fail(HC_ERR_CONFIG, "hc_peer_connect: null argument");
  if (!ctx->peer.region.p || ctx->peer.G != world) return fail(HC_ERR_STATE, "hc_peer_connect: call hc_peer_region(world) first");
  if (rank < 0 || rank >= world) return fail(HC_ERR_CONFIG, "hc_peer_connect: rank %d / world %d", rank, world);
  CUDA_TRY(cudaSetDevice(ctx->device));
  for (void* p : ctx->peer.opened) cudaIpcCloseMemHandle(p);
  ctx->peer.opened.clear();
  for (int q = 0; q < world; ++q) {
    if (q == rank) { ctx->peer.base[q] = ctx->peer.region.p; continue; }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + (size_t)q * 64, 64);
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->peer.opened.push_back(p);
    ctx->peer.base[q] = p;
  }
  return peer_enable(ctx, rank, world);
}
