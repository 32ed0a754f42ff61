// Host rank allocator: PAPER.md Appendix B.1, readings R10-R16.
// Compiled with -ffp-contract=off and without fast-math: every floating-point operation is
// the same IEEE-754 double operation, in the same order, as the oracle, so the plan is
// bit-identical (tests/test_abi_host.py).
#include <algorithm>
#include <cmath>
#include <map>
#include <utility>
#include <vector>

#include "hcinfer.h"
#include "status.h"

namespace {

struct Sal { double phi; int cut; int n; };

// φ_i: σ̂ = σ/σ1; k_j = σ̂_{j-1} − 2σ̂_j + σ̂_{j+1} (interior j); cut = argmax
// (smallest index on ties); S = {1..cut} iff max k > τ; φ = mean_S / mean_R, else 1.
Sal salience(const double* sig, int n, double tau) {
  if (n < 3 || sig[0] == 0.0) return {1.0, 0, n};
  const double s1 = sig[0];
  std::vector<double> hat(n);
  for (int j = 0; j < n; ++j) hat[j] = sig[j] / s1;
  int best_j = -1;
  double best_k = -INFINITY;
  for (int j = 1; j < n - 1; ++j) {
    const double kj = hat[j - 1] - 2.0 * hat[j] + hat[j + 1];
    if (kj > best_k) { best_k = kj; best_j = j; }
  }
  if (!(best_k > tau)) return {1.0, 0, n};
  const int cut = best_j + 1;
  double ss = 0.0, sr = 0.0;
  for (int j = 0; j < cut; ++j) ss = ss + sig[j];
  for (int j = cut; j < n; ++j) sr = sr + sig[j];
  const double mean_s = ss / cut, mean_r = sr / (n - cut);
  return {mean_s / std::max(mean_r, 1e-300), cut, n};
}

std::vector<double> window_normalise(const std::vector<double>& v) {
  double tot = 0.0;
  for (double x : v) tot = tot + x;
  std::vector<double> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = (tot == 0.0) ? 1.0 / (double)v.size() : v[i] / tot;
  return out;
}

// Nearest level, ties up.  Levels stop at 2^62: an rt >= 2^62 returns 2^62, which exceeds every int cap,
// so cap_level maps it to the same level the oracle's unbounded align + cap gives (no overflow, no
// endless loop for huge finite r̃ = 𝒫·r_std).
long long align_rank(double rt, int k0) {
  long long lo = 0, hi = 1LL << k0;
  while (rt >= (double)hi && hi < (1LL << 62)) { lo = hi; hi *= 2; }
  if (rt >= (double)hi) return hi;
  return (rt - (double)lo) < ((double)hi - rt) ? lo : hi;
}

int cap_level(long long r, int cap, int k0) {
  if (r <= cap) return (int)r;
  int lvl = 0;
  long long v = 1LL << k0;
  while (v <= cap) { lvl = (int)v; v *= 2; }
  return lvl;
}

int demote(int r, int k0) { return (r / 2 >= (1 << k0)) ? r / 2 : 0; }

std::vector<double> two_stage(const std::vector<double>& rt, const std::vector<double>& prio,
                              const std::vector<int>& nsal, const std::vector<int>& nall, int mode) {
  const size_t m = rt.size();
  std::vector<double> out(m, 0.0);
  if (mode == 0) {
    for (size_t i = 0; i < m; ++i) {
      const double sal = std::min(rt[i], (double)nsal[i]);
      out[i] = sal + (rt[i] - sal);
    }
    return out;
  }
  double total = 0.0;
  for (double v : rt) total = total + v;
  std::vector<double> caps(m);
  double capsum = 0.0;
  for (size_t i = 0; i < m; ++i) { caps[i] = (double)nsal[i]; capsum = capsum + caps[i]; }
  double rem = std::min(total, capsum);
  std::vector<size_t> active;
  for (size_t i = 0; i < m; ++i) if (caps[i] > 0.0) active.push_back(i);
  while (!active.empty() && rem > 0.0) {
    double psum = 0.0;
    for (size_t i : active) psum = psum + prio[i];
    std::vector<double> w(m, 0.0);
    for (size_t i : active) w[i] = psum > 0.0 ? prio[i] / psum : 1.0 / (double)active.size();
    std::vector<size_t> sat, keep;
    for (size_t i : active) (out[i] + rem * w[i] >= caps[i] ? sat : keep).push_back(i);
    if (sat.empty()) {
      for (size_t i : active) out[i] = out[i] + rem * w[i];
      rem = 0.0;
      break;
    }
    for (size_t i : sat) { rem = rem - (caps[i] - out[i]); out[i] = caps[i]; }
    active = keep;
  }
  if (total > capsum) {
    const double excess = total - capsum;
    std::vector<double> res(m);
    double rsum = 0.0;
    for (size_t i = 0; i < m; ++i) { res[i] = (double)(nall[i] - nsal[i]); rsum = rsum + res[i]; }
    if (rsum > 0.0)
      for (size_t i = 0; i < m; ++i) out[i] = out[i] + excess * res[i] / rsum;
  }
  return out;
}

}  // namespace

extern "C" hc_status hc_allocate_ranks(const hc_sens* recs, int32_t n, const hc_budget* b,
                                       const int32_t* caps, int32_t* ranks_out, double* priority_out) {
  using hc::fail;
  if (!b || n < 0 || (n > 0 && (!recs || !caps || !ranks_out)))
    return fail(HC_ERR_CONFIG, "hc_allocate_ranks: null argument");
  const int L = b->n_layers;
  if (L < 1 || !b->D_layer) return fail(HC_ERR_CONFIG, "hc_allocate_ranks: n_layers < 1 or D_layer null");
  if (b->k0 < 0 || b->k0 > 20) return fail(HC_ERR_CONFIG, "hc_allocate_ranks: k0 out of range");
  if (!(b->top_k_layers >= 1 && b->top_k_layers <= L))
    return fail(HC_ERR_CONFIG, "hc_allocate_ranks: top_k_layers %d out of range [1, %d]", b->top_k_layers, L);
  if (b->two_stage_mode != 0 && b->two_stage_mode != 1) return fail(HC_ERR_CONFIG, "two_stage_mode must be 0 or 1");
  for (int i = 0; i < n; ++i) {
    const hc_sens& r = recs[i];
    if (r.layer < 0 || r.layer >= L || r.window_kind < 0 || r.window_kind > 3)
      return fail(HC_ERR_CONFIG, "record %d: layer/window out of range", i);
    if (!std::isfinite(r.D_matrix) || r.D_matrix < 0.0 || !std::isfinite(r.gate))
      return fail(HC_ERR_NUMERIC, "record %d: non-finite or negative sensitivity", i);
    if (r.sigma && r.n_sigma < 0) return fail(HC_ERR_CONFIG, "record %d: n_sigma < 0", i);
  }
  for (int l = 0; l < L; ++l)
    if (!std::isfinite(b->D_layer[l]) || b->D_layer[l] < 0.0)
      return fail(HC_ERR_NUMERIC, "layer %d: non-finite or negative layer sensitivity", l);
  for (int k = 0; k < 4; ++k)
    if (!std::isfinite(b->r_std[k])) return fail(HC_ERR_NUMERIC, "r_std[%d] not finite", k);

  // φ per record
  std::vector<double> phi(n);
  std::vector<int> nsal(n), nall(n);
  for (int i = 0; i < n; ++i) {
    if (recs[i].sigma) {
      Sal s = salience(recs[i].sigma, recs[i].n_sigma, b->tau);
      phi[i] = s.phi; nsal[i] = s.cut; nall[i] = s.n;
    } else {
      phi[i] = recs[i].phi; nsal[i] = recs[i].n_salient; nall[i] = recs[i].n_total;
    }
  }
  // 𝒮_ℓ: top-K by D (ties: smaller index)
  std::vector<int> order(L);
  for (int l = 0; l < L; ++l) order[l] = l;
  std::stable_sort(order.begin(), order.end(), [&](int a, int c) { return b->D_layer[a] > b->D_layer[c]; });
  std::vector<char> top(L, 0);
  double dmin = INFINITY;
  for (int t = 0; t < b->top_k_layers; ++t) { top[order[t]] = 1; dmin = std::min(dmin, b->D_layer[order[t]]); }
  std::vector<double> S_l(L);
  for (int l = 0; l < L; ++l) S_l[l] = top[l] ? 1.0 : (dmin == 0.0 ? 0.0 : b->D_layer[l] / dmin);

  // windows in first-appearance order (the order is irrelevant: windows are independent)
  std::map<std::pair<int, int>, std::vector<int>> windows;
  for (int i = 0; i < n; ++i) windows[{recs[i].layer, recs[i].window_kind}].push_back(i);

  for (auto& kv : windows) {
    const std::vector<int>& mem = kv.second;
    const int layer = kv.first.first, kind = kv.first.second;
    const size_t m = mem.size();
    std::vector<double> vphi(m), vD(m);
    for (size_t j = 0; j < m; ++j) { vphi[j] = phi[mem[j]]; vD[j] = recs[mem[j]].D_matrix; }
    std::vector<double> V = window_normalise(vphi), S = window_normalise(vD);
    std::vector<double> G(m, 1.0);
    if (b->moe_k > 0) {
      // gates of every slot must be normalised over the activated experts
      std::map<int, double> gsum;
      std::vector<int> slots;
      for (size_t j = 0; j < m; ++j) {
        const int s = recs[mem[j]].slot;
        if (!gsum.count(s)) { gsum[s] = 0.0; slots.push_back(s); }
      }
      for (auto& g : gsum) {
        double t = 0.0;
        for (size_t j = 0; j < m; ++j) if (recs[mem[j]].slot == g.first) t = t + recs[mem[j]].gate;
        if (std::fabs(t - 1.0) > 1e-9) return fail(HC_ERR_NUMERIC, "gates of slot %d do not sum to 1", g.first);
      }
      for (size_t j = 0; j < m; ++j) G[j] = (double)b->moe_k * recs[mem[j]].gate;
    }
    std::vector<double> vs(m);
    for (size_t j = 0; j < m; ++j) vs[j] = V[j] * S[j];
    std::vector<double> P0 = window_normalise(vs), P(m), RT(m);
    const double rstd = b->r_std[kind];
    for (size_t j = 0; j < m; ++j) { P[j] = (G[j] * P0[j]) * S_l[layer]; RT[j] = P[j] * rstd; }
    std::vector<int> ns(m), na(m);
    for (size_t j = 0; j < m; ++j) { ns[j] = nsal[mem[j]]; na[j] = nall[mem[j]]; }
    std::vector<double> RT2 = two_stage(RT, P, ns, na, b->two_stage_mode);
    std::vector<int> r(m);
    for (size_t j = 0; j < m; ++j) r[j] = cap_level(align_rank(RT2[j], b->k0), caps[mem[j]], b->k0);
    // enforce Σ r <= r_std: demote the lowest-𝒫 nonzero member (ties: later member)
    for (;;) {
      long long sum = 0;
      for (int v : r) sum += v;
      if (!((double)sum > rstd)) break;
      int worst = -1;
      for (size_t j = 0; j < m; ++j) {
        if (r[j] <= 0) continue;
        if (worst < 0 || P[j] < P[worst] || (P[j] == P[worst] && (int)j > worst)) worst = (int)j;
      }
      if (worst < 0) break;
      r[worst] = demote(r[worst], b->k0);
    }
    for (size_t j = 0; j < m; ++j) {
      ranks_out[mem[j]] = r[j];
      if (priority_out) priority_out[mem[j]] = P[j];
    }
  }
  return HC_OK;
}
