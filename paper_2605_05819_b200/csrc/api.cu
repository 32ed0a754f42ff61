// C-ABI: context, load_layer (copy + repack), set_rank, compensated_linear (hcinfer.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "decode.h"
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
  std::shared_ptr<DevBuf> rec, U, V;
  int rows() const { return row_end - row_begin; }
  int cap() const { return std::min(std::min(r_stored, N), K); }
};

struct Window {
  int layer = 0, kind = 0, expert = -1;
  std::vector<Member> members;        // sorted by slot
  DevBuf vpart, cnt;                  // launch workspace (self-resetting counters)
  int ws_chunks = -1;
};

using Key = std::tuple<int, int, int>;

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) { cudaGetLastError(); return false; }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

bool admissible_rank(int r) { return r == 0 || (r >= 8 && (r & (r - 1)) == 0); }

}  // namespace

struct hc_ctx {
  int device = 0;
  int sms = 0;
  std::map<Key, Window> windows;
  std::map<std::tuple<int, int, int, int, int>, int> max_ctas;   // (bits, B, K, chunks, vks) -> co-resident CTAs
  DevBuf stage_x, stage_y;
};

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t _e = (expr);                                                                 \
    if (_e != cudaSuccess) return fail(HC_ERR_RUNTIME, "%s: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

extern "C" const char* hc_version(void) { return "hcinfer-b200 0.1 (sm_100a)"; }
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
  *out = c;
  return HC_OK;
}

extern "C" hc_status hc_destroy(hc_ctx* ctx) {
  if (!ctx) return HC_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  delete ctx;
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
  return HC_OK;
}

// copy a host or device source to a device temporary (or return the device pointer)
static const void* to_device(const void* src, size_t bytes, DevBuf& tmp, cudaStream_t st, cudaError_t& err) {
  err = cudaSuccess;
  if (is_device_ptr(src)) return src;
  err = tmp.alloc(bytes);
  if (err != cudaSuccess) return nullptr;
  err = cudaMemcpyAsync(tmp.p, src, bytes, cudaMemcpyHostToDevice, st);
  return tmp.p;
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
  for (int i = 0; i < n_mats; ++i) {
    const hc_matrix_desc& d = mats[i];
    Key key{d.layer, d.window_kind, d.expert};
    Window& w = ctx->windows[key];
    w.layer = d.layer; w.kind = d.window_kind; w.expert = d.expert;
    for (const Member& o : w.members)
      if (o.slot != d.slot && (o.K != d.K || o.bits != d.bits))
        return fail(HC_ERR_CONFIG, "mat %d: window members must share K and bits", i);
    Member m;
    m.slot = d.slot; m.N = d.N; m.K = d.K; m.bits = d.bits; m.r_stored = d.r_stored; m.r_alloc = d.r_alloc;
    m.row_begin = d.row_begin; m.row_end = d.row_end;
    const int rows = m.rows(), G = d.K / hc::kGroup;
    m.rec = std::make_shared<DevBuf>();
    CUDA_TRY(m.rec->alloc((size_t)(rows / hc::kRows) * G * hc::rec_bytes(d.bits)));
    m.U = std::make_shared<DevBuf>();
    m.V = std::make_shared<DevBuf>();
    if (d.r_stored > 0) {
      CUDA_TRY(m.U->alloc((size_t)rows * d.r_stored * 2));
      CUDA_TRY(m.V->alloc((size_t)d.r_stored * d.K * 2));
    }
    DevBuf tc, ts, tz, tu, tv;
    cudaError_t e;
    const uint32_t* codes = (const uint32_t*)to_device(d.codes, (size_t)d.N * d.K * d.bits / 8, tc, st, e);
    CUDA_TRY(e);
    const uint16_t* scales = (const uint16_t*)to_device(d.scales, (size_t)d.N * G * 2, ts, st, e);
    CUDA_TRY(e);
    const uint8_t* zeros = (const uint8_t*)to_device(d.zeros, (size_t)d.N * G, tz, st, e);
    CUDA_TRY(e);
    const uint16_t *U = nullptr, *V = nullptr;
    if (d.r_stored > 0) {
      U = (const uint16_t*)to_device(d.U, (size_t)d.N * d.r_stored * 2, tu, st, e);
      CUDA_TRY(e);
      V = (const uint16_t*)to_device(d.V, (size_t)d.r_stored * d.K * 2, tv, st, e);
      CUDA_TRY(e);
    }
    CUDA_TRY(hc::launch_repack(codes, scales, zeros, U, V, d.K, d.bits, d.r_stored, d.row_begin, rows,
                               (uint8_t*)m.rec->p, (uint32_t*)m.U->p, (uint32_t*)m.V->p, st));
    CUDA_TRY(cudaStreamSynchronize(st));   // temporaries die at scope end
    auto it = std::find_if(w.members.begin(), w.members.end(), [&](const Member& o) { return o.slot == d.slot; });
    if (it != w.members.end()) *it = m; else w.members.push_back(m);
    std::sort(w.members.begin(), w.members.end(), [](const Member& a, const Member& b) { return a.slot < b.slot; });
    if ((int)w.members.size() > hc::kMaxMembers) return fail(HC_ERR_CONFIG, "window has more than %d members", hc::kMaxMembers);
    w.ws_chunks = -1;
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
      return HC_OK;
    }
  return fail(HC_ERR_STATE, "hc_set_rank: slot %d not loaded", slot);
}

extern "C" int64_t hc_window_rows(hc_ctx* ctx, int32_t layer, int32_t kind, int32_t expert) {
  if (!ctx) return -1;
  auto it = ctx->windows.find(Key{layer, kind, expert});
  if (it == ctx->windows.end()) return -1;
  int64_t n = 0;
  for (const Member& m : it->second.members) n += m.rows();
  return n;
}

namespace hc {

// Build the launch arguments of one window (also used by the stack / MoE drivers).
hc_status window_args(hc_ctx* ctx, Window& w, const void* x, int B, void* y, int y_bf16, const void* resid,
                      int ld_resid, DArgs& a, int& grid) {
  std::memset(&a, 0, sizeof(a));
  const Member& m0 = w.members.front();
  a.K = m0.K; a.G = m0.K / kGroup; a.B = B;
  a.x = (const uint16_t*)x; a.y = y; a.y_bf16 = y_bf16;
  a.resid = (const uint16_t*)resid; a.ld_resid = ld_resid;
  int rb = 0, row = 0, chunks = 0, max_chunks = 0;
  a.n_members = (int)w.members.size();
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
    rb += d.n_rb;
    row += m.rows();
    chunks += (m.r_alloc + 15) / 16;
    max_chunks += m.r_stored / 16;
  }
  a.ldy = row;
  a.n_rb = rb;
  a.n_chunks = chunks;
  a.vks = std::max(1, std::min(4, a.G / 8));   // ~8 groups (32 KB of V) per rank-projection item
  if (w.ws_chunks < max_chunks) {
    const int mc = std::max(max_chunks, 1);
    CUDA_TRY(w.vpart.alloc((size_t)mc * kMaxVks * 256 * sizeof(float)));
    CUDA_TRY(w.cnt.alloc(2 * sizeof(unsigned)));
    CUDA_TRY(cudaMemset(w.cnt.p, 0, w.cnt.bytes));
    w.ws_chunks = max_chunks;
  }
  if (a.n_chunks > kMaxChunks) return fail(HC_ERR_CONFIG, "window ranks need %d chunks > %d", a.n_chunks, kMaxChunks);
  static const int dbg = [] { const char* e = getenv("HC_DECODE_DEBUG"); return e ? atoi(e) : 0; }();
  a.dbg = dbg;
  a.vpart = (float*)w.vpart.p;
  a.cnt = (unsigned*)w.cnt.p;
  const auto key = std::make_tuple(m0.bits, B, a.K, a.n_chunks, a.vks);
  auto it = ctx->max_ctas.find(key);
  if (it == ctx->max_ctas.end())
    it = ctx->max_ctas.emplace(key, decode_max_ctas(m0.bits, B, a.K, a.n_chunks, a.vks)).first;
  const int n_items = a.n_chunks * a.vks + a.n_rb;
  static const int per_sm = [] { const char* e = getenv("HC_DECODE_CTAS_PER_SM"); return e ? atoi(e) : 0; }();
  const int cap = per_sm > 0 ? std::min(it->second, per_sm * ctx->sms) : it->second;
  grid = std::max(1, std::min(n_items, cap));
  if (it->second <= 0) return fail(HC_ERR_RUNTIME, "decode kernel cannot be resident on this device");
  return HC_OK;
}

}  // namespace hc

extern "C" hc_status hc_compensated_linear(hc_ctx* ctx, int32_t layer, int32_t kind, int32_t expert,
                                           const void* x, int32_t B, void* y, int32_t y_dtype, void* stream) {
  if (!ctx) return fail(HC_ERR_STATE, "hc_compensated_linear: null context");
  if (B < 1 || B > 16) return fail(HC_ERR_CONFIG, "hc_compensated_linear: B = %d outside [1, 16]", B);
  if (y_dtype != HC_OUT_F32 && y_dtype != HC_OUT_BF16) return fail(HC_ERR_CONFIG, "bad y_dtype %d", y_dtype);
  if (!x || !y) return fail(HC_ERR_CONFIG, "hc_compensated_linear: null x or y");
  auto it = ctx->windows.find(Key{layer, kind, expert});
  if (it == ctx->windows.end() || it->second.members.empty())
    return fail(HC_ERR_STATE, "hc_compensated_linear: window (%d,%d,%d) not loaded", layer, kind, expert);
  CUDA_TRY(cudaSetDevice(ctx->device));
  cudaStream_t st = (cudaStream_t)stream;
  Window& w = it->second;
  const int K = w.members.front().K;
  const int64_t rows = hc_window_rows(ctx, layer, kind, expert);
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
  hc::DArgs a;
  int grid = 0;
  hc_status s = hc::window_args(ctx, w, dx, B, dy, y_dtype == HC_OUT_BF16, nullptr, 0, a, grid);
  if (s != HC_OK) return s;
  CUDA_TRY(hc::launch_decode(a, w.members.front().bits, grid, st));
  if (hy) {
    CUDA_TRY(cudaMemcpyAsync(y, dy, yb, cudaMemcpyDeviceToHost, st));
  }
  if (hx || hy) CUDA_TRY(cudaStreamSynchronize(st));
  return HC_OK;
}
