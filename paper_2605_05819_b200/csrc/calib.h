// GPU calibration: SVD of the quantization error and the salience of its spectrum.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace hc {

struct CalibSvdArgs {
  const float* W;          // device fp32 [n_mats][N][K]: the unquantized weights
  const uint32_t* codes;   // device canonical codes [n_mats][N][K*bits/32]
  const uint16_t* scales;  // device bf16 [n_mats][N][K/group]
  const uint8_t* zeros;    // device u8 [n_mats][N][K/group]
  int n_mats, N, K, bits, group, r;
  double* U;               // device fp64 [n_mats][N][r]    (nullable iff r == 0)
  double* V;               // device fp64 [n_mats][r][K]
  double* sigma;           // device fp64 [n_mats][min(N, K)] (nullable)
  int max_sweeps;
  double tol;              // converged when every pair's |a_p·a_q| / (‖a_p‖‖a_q‖) <= tol
};

size_t calib_workspace_bytes(int n_mats, int N, int K, int r);
cudaError_t calib_svd(const CalibSvdArgs& a, void* workspace, cudaStream_t st, int* sweeps_out);
cudaError_t calib_salience(const double* sigma, int n_mats, int n, double tau, double* phi, int* cut, cudaStream_t st);

}  // namespace hc
