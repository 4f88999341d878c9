// solve.cuh -- (a2) batched code solve, Eq. (somf_alpha) P:592-596:
//   alpha_s = argmin_a 1/2 a^T G a - a^T beta_s + lambda Omega(a)   (s = 1..m)
//
//  (the ridge closed form lives in codes.cuh)
//  k_cd         : cyclic coordinate descent (the paper's solver,
//                 P:1341-1342), one warp per column, maintained gradient
//                 g = beta - G alpha in float64 registers, G packed (upper
//                 triangle, float32) in shared memory so k = 256 fits.
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kSolveThreads = 256;
constexpr int kRidgeMaxK = 160;

__device__ __forceinline__ int packed_off(int i, int k) { return i * k - (i * (i - 1)) / 2; }
template <typename GT>
__device__ __forceinline__ GT packed_get(const GT* P, int i, int j, int k) {
  return i <= j ? P[packed_off(i, k) + (j - i)] : P[packed_off(j, k) + (i - j)];
}

// Cyclic CD, one warp per column; KPL = ceil(k/32) coordinates per lane
// (coordinate j lives in lane j & 31, slot j >> 5).
// GT: the packed Gram's type in shared memory (double when it fits, else float)
template <int KPL, typename GT>
__global__ void __launch_bounds__(kSolveThreads)
k_cd(const double* __restrict__ G, const double* __restrict__ beta, int k, int m,
     double l1, double l2, int positive, double tol, int max_sweeps,
     double* __restrict__ A64, float* __restrict__ A32, int* __restrict__ sweeps_out,
     float* __restrict__ AT32, int ldt, int64_t gstride) {
  // the B-bar kernel may launch now (programmatic dependent launch); it reads
  // the codes only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  // gstride > 0: a Gram per column (estimator (b)); one column per CTA
  G += (int64_t)blockIdx.x * gstride;
  extern __shared__ __align__(16) uint8_t cd_smem[];
  GT* Pk = reinterpret_cast<GT*>(cd_smem);  // packed upper triangle, k(k+1)/2
  const int tid = threadIdx.x, nt = blockDim.x;
  const int np = k * (k + 1) / 2;
  for (int e = tid; e < np; e += nt) {
    // invert packed index: row i with packed_off(i) <= e < packed_off(i+1)
    int i = 0;
    {
      int lo = 0, hi = k - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (packed_off(mid, k) <= e) lo = mid; else hi = mid - 1;
      }
      i = lo;
    }
    const int j = i + (e - packed_off(i, k));
    Pk[e] = (GT)G[(int64_t)i * k + j];
  }
  __syncthreads();
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  for (int s = blockIdx.x * nw + wid; s < m; s += gridDim.x * nw) {
    double alpha[KPL], g[KPL], den[KPL], rden[KPL];
    int roff[KPL];                         // packed_off(row): row's packed segment
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int row = lane + 32 * i;
      alpha[i] = 0.0;
      g[i] = row < k ? beta[(int64_t)row * m + s] : 0.0;
      den[i] = row < k ? (double)packed_get(Pk, row, row, k) + l2 : 1.0;
      rden[i] = den[i] > 0.0 ? 1.0 / den[i] : 0.0;   // off the coordinate chain
      roff[i] = packed_off(row < k ? row : 0, k);
    }
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
      double maxd = 0.0;
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        for (int ol = 0; ol < 32; ++ol) {
          const int j = slot * 32 + ol;
          if (j >= k) break;
          double delta = 0.0;
          if (lane == ol) {
            const double gjj = den[slot] - l2;
            const double z = g[slot] + gjj * alpha[slot];
            double nv;
            if (!(den[slot] > 0.0)) nv = 0.0;                       // R12
            else if (positive) nv = fmax(z - l1, 0.0) * rden[slot];
            else nv = copysign(fmax(fabs(z) - l1, 0.0), z) * rden[slot];
            delta = nv - alpha[slot];
            alpha[slot] = nv;
          }
          delta = __shfl_sync(0xffffffffu, delta, ol);
          if (delta != 0.0) {
            maxd = fmax(maxd, fabs(delta));
            const int joff = packed_off(j, k);
#pragma unroll
            for (int i = 0; i < KPL; ++i) {
              const int row = lane + 32 * i;
              // G[row][j] from the packed upper triangle without index multiplies
              const int a = row <= j ? roff[i] + (j - row) : joff + (row - j);
              if (row < k) g[i] = fma(-(double)Pk[a], delta, g[i]);
            }
          }
        }
      }
      double amax = 0.0;
#pragma unroll
      for (int i = 0; i < KPL; ++i) amax = fmax(amax, fabs(alpha[i]));
      amax = warp_max(amax);
      if (maxd <= tol * fmax(1.0, amax)) { ++sweep; break; }
    }
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int row = lane + 32 * i;
      if (row < k) {
        A64[(int64_t)row * m + s] = alpha[i];
        A32[(int64_t)row * m + s] = (float)alpha[i];
        if (AT32) AT32[(int64_t)s * ldt + row] = (float)alpha[i];
      }
    }
    if (lane == 0 && sweeps_out) atomicMax(sweeps_out, sweep);
  }
}

// Cbar <- (1-w) Cbar + (w/eta) A A^T  (Eq. somf_partial; batch mean R4;
// mode U's coefficients, common.cuh).  32 x 32 tiles of Cbar per CTA, the two
// 32-row panels of the codes staged in shared memory 32 columns at a time
// (coalesced along the batch), 2 x 2 entries per thread; every entry sums
// s = 0 .. eta-1 in order with fma(a_i, a_j, .), so Cbar stays exactly symmetric.
constexpr int kCbT = 32;
__global__ void __launch_bounds__(256)
k_cbar_update(const double* __restrict__ A64, int k, int eta, const double* __restrict__ w_dev,
              double* __restrict__ C64, float* __restrict__ C32) {
  __shared__ double Ai[kCbT][kCbT + 1], Aj[kCbT][kCbT + 1];
  const int i0 = blockIdx.y * kCbT, j0 = blockIdx.x * kCbT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int t0 = 0; t0 < eta; t0 += kCbT) {
    for (int e = threadIdx.x; e < kCbT * kCbT; e += 256) {
      const int r = e / kCbT, c = e % kCbT, t = t0 + c;
      Ai[r][c] = (i0 + r < k && t < eta) ? A64[(int64_t)(i0 + r) * eta + t] : 0.0;
      Aj[r][c] = (j0 + r < k && t < eta) ? A64[(int64_t)(j0 + r) * eta + t] : 0.0;
    }
    __syncthreads();
    const int tn = min(kCbT, eta - t0);
    for (int c = 0; c < tn; ++c) {
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 2; ++v) acc[u][v] = fma(Ai[ty + 16 * u][c], Aj[tx + 16 * v][c], acc[u][v]);
    }
    __syncthreads();
  }
  const double keepd = w_dev[kCoefKeep], gc = w_dev[kCoefGainC];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int i = i0 + ty + 16 * u, j = j0 + tx + 16 * v;
      if (i < k && j < k) {
        const int64_t e = (int64_t)i * k + j;
        const double c = keepd * C64[e] + (gc / eta) * acc[u][v];
        C64[e] = c;
        C32[e] = (float)c;
      }
    }
}

}  // namespace somf
