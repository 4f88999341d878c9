// gemm.cuh -- FFMA tile kernels of the SOMF step (v1: CUDA-core path).
//
//  k_contract   (a1) masked code step, Eq. (a) P:659-660:
//               [beta | G] = r * D_M^T [X_M | D_M], split-K over the q masked
//               rows, rows gathered through the index list (or contiguous).
//  k_contract_reduce  fixed-order float64 sum of the split-K partials.
//  k_bbar_update (a3) Eq. somf_partial: Bbar_M <- (1-w) Bbar_M + w/eta X_M A^T
//  k_residual   (a5) Eq. 3: column sums of (X - D A)^2 over the local rows.
//
// Tiles: 64 x 64 outputs per CTA, 256 threads with 4 x 4 register tiles,
// K-chunk 32 staged in shared memory; loads are warp-contiguous (128 B per
// warp instruction) along the row-major D / X rows.
#pragma once
#include "common.cuh"

namespace somf {

constexpr int TM = 64, TN = 64, TK = 32, kGemmThreads = 256;

// 4x4 micro-tile update from two smem tiles stored [kk][TM+4] / [kk][TN+4].
__device__ __forceinline__ void mma_tile_4x4(const float (*As)[TM + 4], const float (*Bs)[TN + 4],
                                             int ty, int tx, float (&acc)[4][4]) {
#pragma unroll 8
  for (int kk = 0; kk < TK; ++kk) {
    const float4 a = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
    const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
    const float av[4] = {a.x, a.y, a.z, a.w};
    const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
  }
}

// ---------------------------------------------------------------------------
// (a1) partial[split][a][c] = sum_{m in split} D[g_m][a] * Y[m][c],
//      Y[m] = [ X row of m (eta cols) | D[g_m] (k cols) ],  g_m = idx[m] (or m).
// grid = (ceil(k/TM), ceil((eta+k)/TN), nsplit)
// ---------------------------------------------------------------------------
template <bool kGather, bool kXCompact>
__global__ void __launch_bounds__(kGemmThreads)
k_contract(const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev,
           const float* __restrict__ D, int kp, int k,
           const float* __restrict__ X, int64_t ldx, int eta,
           float* __restrict__ partial) {
  __shared__ __align__(16) float As[TK][TM + 4];
  __shared__ __align__(16) float Bs[TK][TN + 4];
  const int nc = eta + k;
  const int a0 = blockIdx.x * TM, c0 = blockIdx.y * TN;
  const int64_t q = *q_dev;
  const int nsplit = gridDim.z, s = blockIdx.z;
  const int64_t m_lo = q * s / nsplit, m_hi = q * (s + 1) / nsplit;
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int lr = tid / 64, lc = tid % 64;     // loader: 4 rows x 64 cols per pass
  float acc[4][4] = {};
  for (int64_t mb = m_lo; mb < m_hi; mb += TK) {
#pragma unroll
    for (int pass = 0; pass < TK / 4; ++pass) {
      const int rr = pass * 4 + lr;
      const int64_t m = mb + rr;
      float av = 0.f, bv = 0.f;
      if (m < m_hi) {
        const int64_t g = kGather ? (int64_t)idx[m] : m;
        const float* drow = D + g * kp;
        const int a = a0 + lc;
        if (a < k) av = drow[a];
        const int c = c0 + lc;
        if (c < eta) {
          const float* xrow = X + (kXCompact ? m : g) * ldx;
          bv = xrow[c];
        } else if (c < nc) {
          bv = drow[c - eta];
        }
      }
      As[rr][lc] = av;
      Bs[rr][lc] = bv;
    }
    __syncthreads();
    mma_tile_4x4(As, Bs, ty, tx, acc);
    __syncthreads();
  }
  float* out = partial + (int64_t)s * k * nc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = a0 + ty * 4 + i;
    if (a >= k) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + tx * 4 + j;
      if (c < nc) out[(int64_t)a * nc + c] = acc[i][j];
    }
  }
}

// Fixed-order float64 reduction of the split-K partials, scaled by r:
// beta (k x eta) and G (k x k), row-major.
__global__ void k_contract_reduce(const float* __restrict__ partial, int nsplit, int k, int eta,
                                  double r, double* __restrict__ beta, double* __restrict__ G) {
  const int nc = eta + k;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)k * nc) return;
  double s = 0.0;
  for (int i = 0; i < nsplit; ++i) s += (double)partial[(int64_t)i * k * nc + e];
  s *= r;
  const int a = (int)(e / nc), c = (int)(e % nc);
  if (c < eta) beta[(int64_t)a * eta + c] = s;
  else G[(int64_t)a * k + (c - eta)] = s;
}

// ---------------------------------------------------------------------------
// (a3) Bbar[g_m][a] = (1-w) Bbar[g_m][a] + (w/eta) sum_s X[m][s] A[a][s]
// rows m in [0, q) (gathered) or all rows (kFull, g = m).  Persistent over
// row tiles: grid = (nrowtiles_launch, ceil(k/TN)).
// ---------------------------------------------------------------------------
template <bool kGather, bool kXCompact>
__global__ void __launch_bounds__(kGemmThreads)
k_bbar_update(const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev,
              const float* __restrict__ X, int64_t ldx, int eta,
              const float* __restrict__ A, int k, float* __restrict__ Bbar, int kp,
              const double* __restrict__ w_dev) {
  __shared__ __align__(16) float Xs[TK][TM + 4];   // [s][row]
  __shared__ __align__(16) float As[TK][TN + 4];   // [s][atom]
  const int64_t q = *q_dev;
  const double keepd = w_dev[kCoefKeep], gb = w_dev[kCoefGainB];
  const float keep = (float)keepd, add = (float)(gb / eta);
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int a0 = blockIdx.y * TN;
  for (int64_t m0 = (int64_t)blockIdx.x * TM; m0 < q; m0 += (int64_t)gridDim.x * TM) {
    float acc[4][4] = {};
    for (int s0 = 0; s0 < eta; s0 += TK) {
      // X tile: 64 rows x 32 s: thread -> (row = tid/4 .. , s-chunk)
#pragma unroll
      for (int pass = 0; pass < (TM * TK) / kGemmThreads; ++pass) {
        const int e = pass * kGemmThreads + tid;
        const int rr = e / TK, ss = e % TK;
        const int64_t m = m0 + rr;
        float v = 0.f;
        if (m < q && s0 + ss < eta) {
          const int64_t g = kGather ? (int64_t)idx[m] : m;
          v = X[(kXCompact ? m : g) * ldx + s0 + ss];
        }
        Xs[ss][rr] = v;
      }
      // A tile: 32 s x 64 atoms (A is k x eta row-major)
#pragma unroll
      for (int pass = 0; pass < (TN * TK) / kGemmThreads; ++pass) {
        const int e = pass * kGemmThreads + tid;
        const int aa = e / TK, ss = e % TK;
        float v = 0.f;
        if (a0 + aa < k && s0 + ss < eta) v = A[(int64_t)(a0 + aa) * eta + s0 + ss];
        As[ss][aa] = v;
      }
      __syncthreads();
      mma_tile_4x4(Xs, As, ty, tx, acc);
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t m = m0 + ty * 4 + i;
      if (m >= q) continue;
      const int64_t g = kGather ? (int64_t)idx[m] : m;
      float* brow = Bbar + g * kp;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int a = a0 + tx * 4 + j;
        if (a < k) brow[a] = fmaf(keep, brow[a], add * acc[i][j]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Mode F (Alg. 3 as printed): P_t^perp Bbar <- (1 - w)
// P_t^perp Bbar + (w / eta) P_t^perp X A^T -- the rows OUTSIDE M_t, which the
// BCD never reads, so this runs on a side stream concurrently with it.  Rows
// in M_t are recognised from the Philox rule itself (R1), no index list; they
// are skipped (the masked-row kernel updates them).  Small footprint (17 KB
// shared, <= 64 registers) so CTAs fit next to the persistent BCD CTAs.
__global__ void __launch_bounds__(kGemmThreads, 4)      // <= 64 registers: fits next to a BCD CTA
k_bbar_comp(const float* __restrict__ X, int64_t ldx, int eta, const float* __restrict__ A, int k,
            float* __restrict__ Bbar, int kp, const double* __restrict__ w_dev, int64_t rows, int64_t row_lo,
            uint64_t seed, const int64_t* __restrict__ t_dev, uint64_t T) {
  __shared__ __align__(16) float Xs[TK][TM + 4];   // [s][row]
  __shared__ __align__(16) float As[TK][TN + 4];   // [s][atom]
  const double keepd = w_dev[kCoefKeep], gb = w_dev[kCoefGainB];
  const uint64_t t = (uint64_t)*t_dev;
  const float keep = (float)keepd, add = (float)(gb / eta);
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int a0 = blockIdx.y * TN;
  for (int64_t m0 = (int64_t)blockIdx.x * TM; m0 < rows; m0 += (int64_t)gridDim.x * TM) {
    float acc[4][4] = {};
    for (int s0 = 0; s0 < eta; s0 += TK) {
#pragma unroll
      for (int pass = 0; pass < (TM * TK) / kGemmThreads; ++pass) {
        const int e = pass * kGemmThreads + tid;
        const int rr = e / TK, ss = e % TK;
        const int64_t m = m0 + rr;
        Xs[ss][rr] = (m < rows && s0 + ss < eta) ? X[m * ldx + s0 + ss] : 0.f;
      }
#pragma unroll
      for (int pass = 0; pass < (TN * TK) / kGemmThreads; ++pass) {
        const int e = pass * kGemmThreads + tid;
        const int aa = e / TK, ss = e % TK;
        As[ss][aa] = (a0 + aa < k && s0 + ss < eta) ? A[(int64_t)(a0 + aa) * eta + s0 + ss] : 0.f;
      }
      __syncthreads();
      mma_tile_4x4(Xs, As, ty, tx, acc);
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t m = m0 + ty * 4 + i;
      if (m >= rows) continue;
      const int64_t grow = row_lo + m;                                  // global row (R1 keys)
      const uint32_t bits = mask_bits(seed, t, grow >> 2, grow & ~3, (grow & ~3) + 4, T);
      if (bits & (1u << (grow & 3))) continue;                         // in M_t: masked kernel
      float* brow = Bbar + m * kp;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int a = a0 + tx * 4 + j;
        if (a < k) brow[a] = fmaf(keep, brow[a], add * acc[i][j]);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// (a5) colsq[c] += sum_i (X[i][c] - sum_a D[i][a] A[a][c])^2 over local rows.
// grid = (row tiles (persistent), ceil(m/TN)).  float64 atomics (objective
// only; not on the per-iteration path).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kGemmThreads)
k_residual(const float* __restrict__ D, int kp, int k, int64_t nrows,
           const float* __restrict__ X, int64_t ldx, int m,
           const float* __restrict__ A, double* __restrict__ colsq) {
  __shared__ __align__(16) float Ds[TK][TM + 4];   // [a][row]
  __shared__ __align__(16) float As[TK][TN + 4];   // [a][col]
  __shared__ double csum[TN];
  const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
  const int c0 = blockIdx.y * TN;
  if (tid < TN) csum[tid] = 0.0;
  for (int64_t r0 = (int64_t)blockIdx.x * TM; r0 < nrows; r0 += (int64_t)gridDim.x * TM) {
    float acc[4][4] = {};
    for (int k0 = 0; k0 < k; k0 += TK) {
#pragma unroll
      for (int pass = 0; pass < (TM * TK) / kGemmThreads; ++pass) {
        const int e = pass * kGemmThreads + tid;
        const int rr = e / TK, aa = e % TK;
        float v = 0.f;
        if (r0 + rr < nrows && k0 + aa < k) v = D[(r0 + rr) * kp + k0 + aa];
        Ds[aa][rr] = v;
      }
#pragma unroll
      for (int pass = 0; pass < (TN * TK) / kGemmThreads; ++pass) {
        const int e = pass * kGemmThreads + tid;
        const int aa = e / TN, cc = e % TN;
        float v = 0.f;
        if (k0 + aa < k && c0 + cc < m) v = A[(int64_t)(k0 + aa) * m + c0 + cc];
        As[aa][cc] = v;
      }
      __syncthreads();
      mma_tile_4x4(Ds, As, ty, tx, acc);
      __syncthreads();
    }
    double part[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t row = r0 + ty * 4 + i;
      if (row >= nrows) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + tx * 4 + j;
        if (c < m) {
          const double d = (double)X[row * ldx + c] - (double)acc[i][j];
          part[j] += d * d;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) atomicAdd(&csum[tx * 4 + j], part[j]);
  }
  __syncthreads();
  if (tid < TN && c0 + tid < m) atomicAdd(&colsq[c0 + tid], csum[tid]);
}

}  // namespace somf
