// GPU calibration side: the factors of the quantization error and the allocator's
// spectrum input, computed on the device in float64.
//
//   ΔW = W − deq(W_q)                          ("XΔW ≈ (XA_r)B_r")
//   ΔW = P·diag(σ)·Qᵀ (SVD)                    (A_r, B_r "obtained from the SVD of ΔW")
//   U = P[:, :r],  V = diag(σ[:r])·Q[:, :r]ᵀ   (R4, the north_star orientation y = Ŵx + U(Vx))
//   φ = salience of σ                           (App. B.1 eq. A8; R10)
//
// SVD: one-sided (Hestenes) Jacobi on the columns of ΔW (or of ΔWᵀ when K > N: the shorter side is the
// column count), float64, round-robin ("circle") ordering: every step rotates K/2 disjoint column pairs,
// one CTA per pair, so a step is one launch over all pairs of all matrices of the batch.  A sweep is C − 1
// steps; sweeps repeat until every pair's |a_p·a_q| / (‖a_p‖‖a_q‖) is below 1e-15 (measured per sweep with an
// atomicMax on the bit pattern of a non-negative double).  The orthogonalised columns give σ (their
// norms) and one side of the factorisation directly; the other side is one float64 GEMM against a copy of
// ΔW.  Reductions are fixed-order (warp shuffle tree, then warps in order): the result is deterministic.
// Not on the hot path (offline calibration); the hot path consumes U, V after hc_load_layer.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include <cstring>
#include <vector>

#include "calib.h"

namespace hc {

namespace {

constexpr int kCalThreads = 256;

__device__ __forceinline__ double bf16_to_f64(uint16_t b) { return (double)__uint_as_float((uint32_t)b << 16); }

// Code q of element k of one row of a canonical code stream (hcinfer.h: element k at bits [b·k, b·k + b)).
__device__ __forceinline__ unsigned code_at(const uint32_t* row, int k, int bits) {
  const long long bit = (long long)bits * k;
  const int w = (int)(bit >> 5), o = (int)(bit & 31);
  unsigned long long v = row[w];
  if (o + bits > 32) v |= (unsigned long long)row[w + 1] << 32;
  return (unsigned)((v >> o) & ((1u << bits) - 1u));
}

// Fixed-order block sum of three doubles (256 threads): warp trees, then the 8 warp partials in order.
__device__ __forceinline__ void block_sum3(double& a, double& b, double& c, double* sh /* [3][8] */) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
    b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
    c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sh[w] = a; sh[8 + w] = b; sh[16 + w] = c; }
  __syncthreads();
  a = 0.0; b = 0.0; c = 0.0;
  for (int i = 0; i < kCalThreads / 32; ++i) { a += sh[i]; b += sh[8 + i]; c += sh[16 + i]; }
  __syncthreads();
}

// ΔW into the column store A[m][c][l] (column c contiguous, length L) and its copy D.  trans = 0: columns
// are ΔW's columns (C = K, L = N); trans = 1: columns are ΔW's rows (C = N, L = K).  ΔW = W − s·(q − z):
// s·(q − z) is exact in float64, the subtraction rounds once (as the oracle's float64 W − Ŵ).
__global__ void delta_kernel(const float* __restrict__ W, const uint32_t* __restrict__ codes,
                             const uint16_t* __restrict__ scales, const uint8_t* __restrict__ zeros, int N, int K,
                             int bits, int group, int trans, double* __restrict__ A, double* __restrict__ D) {
  __shared__ double t[32][33];
  const int m = blockIdx.z, i0 = blockIdx.y * 32, j0 = blockIdx.x * 32;   // tile of rows i, cols j of ΔW
  const int tx = threadIdx.x, ty = threadIdx.y;                            // 32 x 8
  const int G = K / group, words = K * bits / 32;
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    const size_t row = (size_t)m * N + i;
    const double s = bf16_to_f64(scales[row * G + j / group]);
    const double z = (double)zeros[row * G + j / group];
    const double q = (double)code_at(codes + row * words, j, bits);
    t[r][tx] = (double)W[row * K + j] - s * (q - z);
  }
  __syncthreads();
  const size_t base = (size_t)m * N * K;
  if (trans) {   // A[i][j] (row i of ΔW is column i, contiguous in j): write the tile as read
    for (int r = ty; r < 32; r += 8) {
      const size_t o = base + (size_t)(i0 + r) * K + j0 + tx;
      A[o] = t[r][tx];
      D[o] = t[r][tx];
    }
  } else {       // A[j][i] (column j of ΔW contiguous in i): transpose through the tile
    for (int r = ty; r < 32; r += 8) {
      const size_t o = base + (size_t)(j0 + r) * N + i0 + tx;
      A[o] = t[tx][r];
      D[o] = t[tx][r];
    }
  }
}

// One round-robin step: pair p of the circle ordering at `step` (position 0 fixed, the others rotate).
__device__ __forceinline__ int circle_col(int pos, int step, int C) { return pos == 0 ? 0 : 1 + (pos - 1 + step) % (C - 1); }

__global__ void __launch_bounds__(kCalThreads) jacobi_step_kernel(double* __restrict__ A, int C, int L, int step,
                                                                  unsigned long long* __restrict__ off) {
  __shared__ double sh[24];
  __shared__ double rot[3];   // c, s, apply
  const int m = blockIdx.y, pr = blockIdx.x;
  const int p = circle_col(pr, step, C), q = circle_col(C - 1 - pr, step, C);
  double* ap = A + ((size_t)m * C + p) * L;
  double* aq = A + ((size_t)m * C + q) * L;
  double al = 0.0, be = 0.0, ga = 0.0;
  for (int i = threadIdx.x; i < L; i += kCalThreads) {
    const double x = ap[i], y = aq[i];
    al = fma(x, x, al);
    be = fma(y, y, be);
    ga = fma(x, y, ga);
  }
  block_sum3(al, be, ga, sh);
  if (threadIdx.x == 0) {
    double c = 1.0, s = 0.0, apply = 0.0;
    const double nrm = sqrt(al) * sqrt(be);
    if (ga != 0.0 && nrm > 0.0) {
      const double o = fabs(ga) / nrm;
      atomicMax(off + m, (unsigned long long)__double_as_longlong(o));
      if (o > 1e-17) {
        // Rutishauser: ζ = (β − α) / 2γ, t = sign(ζ) / (|ζ| + √(1 + ζ²)), c = 1/√(1 + t²), s = c·t
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        c = 1.0 / sqrt(1.0 + t * t);
        s = c * t;
        apply = 1.0;
      }
    }
    rot[0] = c; rot[1] = s; rot[2] = apply;
  }
  __syncthreads();
  if (rot[2] == 0.0) return;
  const double c = rot[0], s = rot[1];
  for (int i = threadIdx.x; i < L; i += kCalThreads) {
    const double x = ap[i], y = aq[i];
    ap[i] = c * x - s * y;
    aq[i] = s * x + c * y;
  }
}

// σ_c = ‖a_c‖ (fixed-order block sum), one CTA per column.
__global__ void __launch_bounds__(kCalThreads) norms_kernel(const double* __restrict__ A, int C, int L,
                                                            double* __restrict__ nrm) {
  __shared__ double sh[24];
  const int m = blockIdx.y, c = blockIdx.x;
  const double* a = A + ((size_t)m * C + c) * L;
  double s = 0.0, d1 = 0.0, d2 = 0.0;
  for (int i = threadIdx.x; i < L; i += kCalThreads) s = fma(a[i], a[i], s);
  block_sum3(s, d1, d2, sh);
  if (threadIdx.x == 0) nrm[(size_t)m * C + c] = sqrt(s);
}

// Sort descending by counting (ties: smaller column first): perm[m][rank] = column, sigma[m][rank] = σ.
__global__ void rank_kernel(const double* __restrict__ nrm, int C, int* __restrict__ perm, double* __restrict__ sigma) {
  const int m = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double* v = nrm + (size_t)m * C;
  const double x = v[c];
  int rk = 0;
  for (int i = 0; i < C; ++i) rk += (v[i] > x) || (v[i] == x && i < c);
  perm[(size_t)m * C + rk] = c;
  sigma[(size_t)m * C + rk] = x;
}

// X[m][j][l] = a_{perm j}[l] / σ_j for j < r (0 when σ_j = 0).
__global__ void unit_kernel(const double* __restrict__ A, const int* __restrict__ perm, const double* __restrict__ sigma,
                            int C, int L, int r, double* __restrict__ X) {
  const int m = blockIdx.z, j = blockIdx.y, l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const double sg = sigma[(size_t)m * C + j];
  const double v = A[((size_t)m * C + perm[(size_t)m * C + j]) * L + l];
  X[((size_t)m * r + j) * L + l] = sg > 0.0 ? v / sg : 0.0;
}

// Y[m][c][j] = Σ_l D[m][c][l] · X[m][j][l]  (float64, 16 x 16 output tiles, fixed l order).
__global__ void gemm_dx_kernel(const double* __restrict__ D, const double* __restrict__ X, int C, int L, int r,
                               double* __restrict__ Y) {
  __shared__ double sd[16][17], sx[16][17];
  const int m = blockIdx.z, c0 = blockIdx.y * 16, j0 = blockIdx.x * 16;
  const int tx = threadIdx.x, ty = threadIdx.y;   // 16 x 16: tx = j, ty = c
  double acc = 0.0;
  for (int l0 = 0; l0 < L; l0 += 16) {
    const int l = l0 + tx;
    sd[ty][tx] = (c0 + ty < C && l < L) ? D[((size_t)m * C + c0 + ty) * L + l] : 0.0;
    sx[ty][tx] = (j0 + ty < r && l < L) ? X[((size_t)m * r + j0 + ty) * L + l] : 0.0;
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) acc = fma(sd[ty][kk], sx[tx][kk], acc);
    __syncthreads();
  }
  if (c0 + ty < C && j0 + tx < r) Y[((size_t)m * C + c0 + ty) * r + j0 + tx] = acc;
}

// Assemble U [m][N][r] and V [m][r][K] with the sign convention (first nonzero entry of each U column >= 0,
// DESIGN.md R5), one CTA per (matrix, rank j).
//   trans = 0: U[:, j] = X[j] (the unit columns, length N), V[j][k] = Y[k][j]
//   trans = 1: U[i][j] = Y[i][j] / σ_j,                   V[j][k] = σ_j·X[j][k]
__global__ void __launch_bounds__(kCalThreads) assemble_kernel(const double* __restrict__ X, const double* __restrict__ Y,
                                                               const double* __restrict__ sigma, int N, int K, int C,
                                                               int r, int trans, double* __restrict__ U,
                                                               double* __restrict__ V) {
  __shared__ int first;
  const int m = blockIdx.y, j = blockIdx.x;
  const double sg = sigma[(size_t)m * C + j];
  auto u_at = [&](int i) -> double {
    return trans ? (sg > 0.0 ? Y[((size_t)m * C + i) * r + j] / sg : 0.0) : X[((size_t)m * r + j) * N + i];
  };
  if (threadIdx.x == 0) first = N;
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += kCalThreads)
    if (u_at(i) != 0.0) atomicMin(&first, i);
  __syncthreads();
  const double sgn = (first < N && u_at(first) < 0.0) ? -1.0 : 1.0;
  for (int i = threadIdx.x; i < N; i += kCalThreads) U[((size_t)m * N + i) * r + j] = sgn * u_at(i);
  for (int k = threadIdx.x; k < K; k += kCalThreads) {
    const double v = trans ? sg * X[((size_t)m * r + j) * K + k] : Y[((size_t)m * C + k) * r + j];
    V[((size_t)m * r + j) * K + k] = sgn * v;
  }
}

// Salience φ (R10), one thread per spectrum: the oracle's float64 operations in its order, with
// explicit round-to-nearest intrinsics so that no multiply-add is contracted (bit-exact given the same σ).
__global__ void salience_kernel(const double* __restrict__ sigma, int n_mats, int n, double tau,
                                double* __restrict__ phi, int* __restrict__ cut_out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n_mats) return;
  const double* sg = sigma + (size_t)m * n;
  if (n < 3 || sg[0] == 0.0) { phi[m] = 1.0; cut_out[m] = 0; return; }
  const double s1 = sg[0];
  int best_j = -1;
  double best_k = -INFINITY;
  for (int j = 1; j < n - 1; ++j) {
    const double h0 = __ddiv_rn(sg[j - 1], s1), h1 = __ddiv_rn(sg[j], s1), h2 = __ddiv_rn(sg[j + 1], s1);
    const double kj = __dadd_rn(__dsub_rn(h0, __dmul_rn(2.0, h1)), h2);
    if (kj > best_k) { best_k = kj; best_j = j; }
  }
  if (!(best_k > tau)) { phi[m] = 1.0; cut_out[m] = 0; return; }
  const int cut = best_j + 1;
  double ss = 0.0, sr = 0.0;
  for (int j = 0; j < cut; ++j) ss = __dadd_rn(ss, sg[j]);
  for (int j = cut; j < n; ++j) sr = __dadd_rn(sr, sg[j]);
  const double mean_s = __ddiv_rn(ss, (double)cut), mean_r = __ddiv_rn(sr, (double)(n - cut));
  phi[m] = __ddiv_rn(mean_s, fmax(mean_r, 1e-300));
  cut_out[m] = cut;
}

}  // namespace

size_t calib_workspace_bytes(int n_mats, int N, int K, int r) {
  const size_t C = (size_t)(K <= N ? K : N), L = (size_t)(K <= N ? N : K);
  const size_t a = (size_t)n_mats * C * L * sizeof(double);
  return 2 * a                                           // A, D
         + (size_t)n_mats * C * (2 * sizeof(double) + sizeof(int))   // norms, sorted σ, perm
         + (size_t)n_mats * r * L * sizeof(double)       // X
         + (size_t)n_mats * C * r * sizeof(double)       // Y
         + (size_t)n_mats * sizeof(unsigned long long) + 256;
}

cudaError_t calib_svd(const CalibSvdArgs& g, void* ws, cudaStream_t st, int* sweeps_out) {
  const int trans = g.K > g.N ? 1 : 0;
  const int C = trans ? g.N : g.K, L = trans ? g.K : g.N;
  uint8_t* p = (uint8_t*)ws;
  auto take = [&](size_t b) { uint8_t* q = p; p += (b + 255) & ~(size_t)255; return q; };
  double* A = (double*)take((size_t)g.n_mats * C * L * sizeof(double));
  double* D = (double*)take((size_t)g.n_mats * C * L * sizeof(double));
  double* nrm = (double*)take((size_t)g.n_mats * C * sizeof(double));
  double* sig = (double*)take((size_t)g.n_mats * C * sizeof(double));
  int* perm = (int*)take((size_t)g.n_mats * C * sizeof(int));
  double* X = (double*)take((size_t)g.n_mats * (g.r > 0 ? g.r : 1) * L * sizeof(double));
  double* Y = (double*)take((size_t)g.n_mats * C * (g.r > 0 ? g.r : 1) * sizeof(double));
  unsigned long long* off = (unsigned long long*)take((size_t)g.n_mats * sizeof(unsigned long long));

  delta_kernel<<<dim3(g.K / 32, g.N / 32, g.n_mats), dim3(32, 8), 0, st>>>(g.W, g.codes, g.scales, g.zeros, g.N, g.K,
                                                                           g.bits, g.group, trans, A, D);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  std::vector<unsigned long long> h(g.n_mats);
  int sweeps = 0;
  for (; sweeps < g.max_sweeps; ++sweeps) {
    if ((e = cudaMemsetAsync(off, 0, (size_t)g.n_mats * sizeof(unsigned long long), st)) != cudaSuccess) return e;
    for (int s = 0; s < C - 1; ++s)
      jacobi_step_kernel<<<dim3(C / 2, g.n_mats), kCalThreads, 0, st>>>(A, C, L, s, off);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(h.data(), off, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    double worst = 0.0;
    for (unsigned long long v : h) {
      double d;
      memcpy(&d, &v, sizeof(d));
      worst = d > worst ? d : worst;
    }
    if (worst <= g.tol) { ++sweeps; break; }
  }
  if (sweeps_out) *sweeps_out = sweeps;
  norms_kernel<<<dim3(C, g.n_mats), kCalThreads, 0, st>>>(A, C, L, nrm);
  rank_kernel<<<dim3((C + 255) / 256, g.n_mats), 256, 0, st>>>(nrm, C, perm, sig);
  if (g.sigma) {
    const int ns = C;   // min(N, K) singular values
    if ((e = cudaMemcpyAsync(g.sigma, sig, (size_t)g.n_mats * ns * sizeof(double), cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
  }
  if (g.r > 0) {
    unit_kernel<<<dim3((L + 255) / 256, g.r, g.n_mats), 256, 0, st>>>(A, perm, sig, C, L, g.r, X);
    gemm_dx_kernel<<<dim3((g.r + 15) / 16, (C + 15) / 16, g.n_mats), dim3(16, 16), 0, st>>>(D, X, C, L, g.r, Y);
    assemble_kernel<<<dim3(g.r, g.n_mats), kCalThreads, 0, st>>>(X, Y, sig, g.N, g.K, C, g.r, trans, g.U, g.V);
  }
  return cudaGetLastError();
}

cudaError_t calib_salience(const double* sigma, int n_mats, int n, double tau, double* phi, int* cut, cudaStream_t st) {
  salience_kernel<<<(n_mats + 127) / 128, 128, 0, st>>>(sigma, n_mats, n, tau, phi, cut);
  return cudaGetLastError();
}

}  // namespace hc
