// estimators.cuh -- the code-step estimators (b) and (c) of PAPER.md §III-B
// (Table I) on top of the masked contraction of estimator (a):
//
//  k_est_average : per column s of the batch, sample i = ids[s]:
//                    c^(i) += 1, gamma = c^(i)^-v
//                    beta^(i) <- (1 - gamma) beta^(i) + gamma r D^T M_t x^(i)
//                    (b) G^(i) <- (1 - gamma) G^(i) + gamma r D^T M_t D
//                  and the batch's estimates beta (k x eta) [and G per column].
//                  Reading R23: Alg. 3's "(1 - gamma) G^(i)_{t-1}" in the beta
//                  line is beta^(i)_{t-1}; c = 1 gives gamma = 1 (overwrite).
//                  Reading R25: the ids of a batch are distinct; a repeat is
//                  detected through a per-sample stamp (last iteration seen)
//                  and flagged (err = 8).
//  k_gex_update  : (c) the exact Gram D_t^T D_t from D_{t-1}^T D_{t-1}: only
//                  the masked rows changed in Alg. 4
//                    G <- G - P_t D_old^T P_t D_old + P_t D_new^T P_t D_new
//                  with P_t D_old^T P_t D_old = G_masked / r of this step's
//                  contraction and P_t D_new^T P_t D_new a second contraction
//                  of the updated rows.
// All statistics in fp64.
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kEstThreads = 256;

__global__ void __launch_bounds__(kEstThreads)
k_est_average(const int64_t* __restrict__ ids, int64_t n, const double* __restrict__ beta_m,
              const double* __restrict__ G_m, int k, int eta, double v, const int64_t* __restrict__ t_dev,
              int* __restrict__ cnt, int* __restrict__ stamp, double* __restrict__ bcache,
              double* __restrict__ gcache, double* __restrict__ beta_out, double* __restrict__ G_out,
              int* __restrict__ err) {
  __shared__ double gam_s;
  __shared__ int64_t i_s;
  const int s = blockIdx.x, tid = threadIdx.x;
  if (tid == 0) {
    const int64_t i = ids[s];
    double gam = 0.0;
    if (i < 0 || i >= n) {
      atomicExch(err, 7);
      i_s = -1;
    } else {
      const int t = (int)*t_dev;
      if (atomicExch(stamp + i, t) == t) atomicExch(err, 8);        // R25: repeated id in one batch
      const int c = atomicAdd(cnt + i, 1) + 1;
      gam = pow((double)c, -v);                                     // gamma_c = c^-v
      i_s = i;
    }
    gam_s = gam;
  }
  __syncthreads();
  const int64_t i = i_s;
  if (i < 0) return;
  const double gam = gam_s, keep = 1.0 - gam;
  for (int j = tid; j < k; j += kEstThreads) {
    double* bc = bcache + i * k + j;
    const double b = keep == 0.0 ? beta_m[(int64_t)j * eta + s] : fma(keep, *bc, gam * beta_m[(int64_t)j * eta + s]);
    *bc = b;
    beta_out[(int64_t)j * eta + s] = b;
  }
  if (gcache) {
    const int64_t kk = (int64_t)k * k;
    for (int64_t e = tid; e < kk; e += kEstThreads) {
      double* gc = gcache + i * kk + e;
      const double g = keep == 0.0 ? G_m[e] : fma(keep, *gc, gam * G_m[e]);
      *gc = g;
      G_out[(int64_t)s * kk + e] = g;
    }
  }
}

// G_ex += G_new - G_m / r   (k x k, fp64)
__global__ void k_gex_update(double* __restrict__ G_ex, const double* __restrict__ G_m,
                             const double* __restrict__ G_new, int kk, double inv_r) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < kk) G_ex[e] = G_ex[e] + (G_new[e] - G_m[e] * inv_r);
}

__global__ void k_copy_f64(double* __restrict__ dst, const double* __restrict__ src, int n) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) dst[e] = src[e];
}

}  // namespace somf
