// codes.cuh -- (a2) ridge codes and (a3) Cbar:
//
//  k_ridge_codes<KPL> : alpha = (G + lambda I)^-1 beta  (Eq. somf_alpha,
//                  P:592-596, nu = 1, no positivity), k <= 32 KPL <= 160.
//                  Every CTA factorises G + lambda I redundantly in shared
//                  memory (fp64 blocked LL^T, 8-column panels, each diagonal
//                  block and its inverse in registers; v3 below), then each
//                  warp solves one right-hand side with 8 x 8 block
//                  mat-vecs through the stored block inverses.  Each CTA
//                  also writes its partial sum_s alpha_s alpha_s^T for the
//                  Cbar update.
//  k_cbar_finalize : Cbar <- (1 - w) Cbar + (w / eta) sum_b partial_b
//                  (Eq. somf_partial, batch mean R4), partials added in
//                  block order (deterministic).
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kRcThreads = 256;
constexpr int kRcMaxK = 160;

// 1/sqrt(d) in fp64: fp32 MUFU estimate + two Newton steps (rel. error ~1e-16),
// ~3x shorter latency than sqrt() followed by a division
__device__ __forceinline__ double rc_rsqrt(double d) {
  double y = (double)rsqrtf((float)d);
  y = y * fma(-0.5 * d, y * y, 1.5);
  y = y * fma(-0.5 * d, y * y, 1.5);
  return y;
}

template <int KPL>
__device__ __forceinline__ double rc_pick(const double (&y)[KPL], int c) {
  double v = 0.0;
#pragma unroll
  for (int i = 0; i < KPL; ++i)
    if (i == c) v = y[i];
  return v;
}

// ---------------------------------------------------------------------------
// v3: blocked LL^T with 8-column panels, every panel's diagonal block and its
// inverse in registers, no serial chain outside the 8 x 8 blocks.
//
// Per panel jb (K = k rounded up to 8, identity padding):
//   1. every thread factorises the 8 x 8 diagonal block A_bb = L_bb L_bb^T in
//      registers (fp32 rsqrt seed + two fp64 Newton steps per pivot) and forms
//      W_b = L_bb^-1 (8 x 8 lower triangular) -- redundantly, so no barrier;
//   2. panel rows i >= jb + 8 (one thread per row): L_i,b = A_i,b W_b^T (a
//      mat-vec with the inverse: 64 independent FMAs, no chain);
//   3. barrier; rank-8 trailing update of the lower triangle, every thread a
//      strided share of the entries (the panel row of i kept in registers);
//      barrier.
// W_b of every block is kept in shared memory, so the substitutions are 8 x 8
// mat-vecs per block too: one warp per right-hand side, lane l holding rows
// l, l + 32, ...; per block the 8 entries are broadcast by shuffles,
// multiplied by W_b (forward) or W_b^T (backward), and the other rows updated.
// ---------------------------------------------------------------------------
constexpr int kRcB = 8;

// smem doubles: K (K + 1) (L, lower) + (K / 8) 64 (W_b) + 8 K (codes of the 8 warps)
__host__ __device__ constexpr size_t rc_smem_doubles(int K) {
  return (size_t)K * (K + 1) + (size_t)(K / kRcB) * kRcB * kRcB + (size_t)8 * K;
}

template <int KPL>
__global__ void __launch_bounds__(kRcThreads)
k_ridge_codes(const double* __restrict__ G, const double* __restrict__ beta, int k, int m, double lam,
              double* __restrict__ A64, float* __restrict__ A32, float* __restrict__ AT32, int ldt,
              double* __restrict__ cpart, int* __restrict__ err, long long* __restrict__ prof,
              int64_t gstride, int cpc) {
  // the B-bar kernel may launch now (programmatic dependent launch); it reads
  // the codes only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  // gstride > 0: a Gram per column (estimator (b)); cpc columns per CTA (8, or 1)
  G += (int64_t)blockIdx.x * gstride;
  extern __shared__ double rc_smem[];
  long long t_mark = clock64();
#define RC_MARK(slot)                                                     \
  do {                                                                    \
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {                    \
      const long long now_ = clock64();                                   \
      prof[slot] += now_ - t_mark;                                        \
      t_mark = now_;                                                      \
    }                                                                     \
  } while (0)
  const int kr = k;
  const int K = (k + kRcB - 1) & ~(kRcB - 1);
  const int ld = K + 1;
  double* M = rc_smem;                              // K x ld, lower triangle
  double* Wb = M + (size_t)K * ld;                  // (K / 8) x 64
  double* Y = Wb + (size_t)(K / kRcB) * 64;         // 8 x K
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // ---- load G + lambda I (lower triangle, identity padding), up to kRcLd
  // entries per thread in flight (k = 70: all 21 of a thread, one L2 round
  // trip; only the j <= i half actually loads)
  constexpr int kRcLd = 21;
  for (int e0 = tid; e0 < K * K; e0 += kRcLd * kRcThreads) {
    double g[kRcLd];
#pragma unroll
    for (int u = 0; u < kRcLd; ++u) {
      const int e = e0 + u * kRcThreads;
      const int i = e / K, j = e % K;
      g[u] = (e < K * K && j <= i && i < kr && j < kr) ? __ldg(G + (int64_t)i * kr + j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kRcLd; ++u) {
      const int e = e0 + u * kRcThreads;
      const int i = e / K, j = e % K;
      if (e < K * K && j <= i) M[i * ld + j] = (i < kr && j < kr) ? g[u] + (i == j ? lam : 0.0) : (i == j ? 1.0 : 0.0);
    }
  }
  __syncthreads();
  RC_MARK(0);
  bool bad = false;
  // warp 0: factorise the (already updated) 8 x 8 diagonal block at jb, every
  // lane redundantly in registers; lane 0..63 entries written back: L_bb into
  // M, W_b = L_bb^-1 into Wb.  `pre` (optional) first applies the rank-8
  // update of the previous panel (columns pb..pb+7) to the block (lookahead).
  auto diag_block = [&](int jb, int pb) {
    double L[kRcB][kRcB], W[kRcB][kRcB];
#pragma unroll
    for (int a = 0; a < kRcB; ++a)
#pragma unroll
      for (int c = 0; c < kRcB; ++c) L[a][c] = c <= a ? M[(jb + a) * ld + jb + c] : 0.0;
    if (pb >= 0) {
      double P[kRcB][kRcB];
#pragma unroll
      for (int a = 0; a < kRcB; ++a)
#pragma unroll
        for (int u = 0; u < kRcB; ++u) P[a][u] = M[(jb + a) * ld + pb + u];
#pragma unroll
      for (int a = 0; a < kRcB; ++a)
#pragma unroll
        for (int c = 0; c <= a; ++c) {
          double v = L[a][c];
#pragma unroll
          for (int u = 0; u < kRcB; ++u) v = fma(-P[a][u], P[c][u], v);
          L[a][c] = v;
        }
    }
#pragma unroll
    for (int c = 0; c < kRcB; ++c) {
      const double d = L[c][c];
      bad |= !(d > 0.0);
      double ir = 0.0;
      if (d > 0.0) {
        // fp32 seed + one fp64 Newton step: relative error ~1e-14
        ir = (double)rsqrtf((float)d);
        ir = ir * fma(-0.5 * d, ir * ir, 1.5);
      }
      L[c][c] = d * ir;
      W[c][c] = ir;                                 // 1 / L_cc
#pragma unroll
      for (int a2 = c + 1; a2 < kRcB; ++a2) L[a2][c] *= ir;
#pragma unroll
      for (int a2 = c + 1; a2 < kRcB; ++a2)
#pragma unroll
        for (int b2 = c + 1; b2 <= a2; ++b2) L[a2][b2] = fma(-L[a2][c], L[b2][c], L[a2][b2]);
    }
#pragma unroll
    for (int c = 0; c < kRcB; ++c) {
#pragma unroll
      for (int i = c + 1; i < kRcB; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int l = c; l < i; ++l) acc = fma(L[i][l], W[l][c], acc);
        W[i][c] = -W[i][i] * acc;
      }
#pragma unroll
      for (int i = 0; i < c; ++i) W[i][c] = 0.0;
    }
#pragma unroll
    for (int h2 = 0; h2 < 2; ++h2) {
      const int e = lane + 32 * h2, a2 = e / kRcB, c2 = e % kRcB;
      double lv = 0.0, wv = 0.0;
#pragma unroll
      for (int a3 = 0; a3 < kRcB; ++a3)
#pragma unroll
        for (int c3 = 0; c3 < kRcB; ++c3)
          if (a3 == a2 && c3 == c2) { lv = L[a3][c3]; wv = W[a3][c3]; }
      if (c2 <= a2) M[(jb + a2) * ld + jb + c2] = lv;
      Wb[(jb / kRcB) * 64 + e] = wv;
    }
  };
  if (wid == 0) diag_block(0, -1);
  __syncthreads();
  for (int jb = 0; jb < K; jb += kRcB) {
    // ---- panel rows below: L_i,b = A_i,b W_b^T (W_b lower triangular) ------
    const double* w = Wb + (jb / kRcB) * 64;
    for (int i = jb + kRcB + tid; i < K; i += kRcThreads) {
      double x[kRcB];
#pragma unroll
      for (int u = 0; u < kRcB; ++u) x[u] = M[i * ld + jb + u];
#pragma unroll
      for (int t = 0; t < kRcB; ++t) {
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u <= t; ++u) acc = fma(x[u], w[t * kRcB + u], acc);
        M[i * ld + jb + t] = acc;
      }
    }
    __syncthreads();
    const int jn = jb + kRcB, n = K - jn;
    if (n > 0) {
      if (wid == 0) {
        // lookahead: the next diagonal block, updated by this panel and factorised
        diag_block(jn, jb);
      } else {
        // rank-8 trailing update of the lower triangle below the panel, the
        // next diagonal block excepted (warp 0 owns it): warps 1..7, thread
        // (ty, tx) rows jn + ty + 14 s, columns jn + tx + 16 c
        const int t2 = tid - 32, ty = t2 >> 4, tx = t2 & 15;
        constexpr int NY = (kRcThreads - 32) / 16;
        for (int ii = ty; ii < n; ii += NY) {
          const int i = jn + ii;
          double li[kRcB];
#pragma unroll
          for (int u = 0; u < kRcB; ++u) li[u] = M[i * ld + jb + u];
          for (int ll = (ii < kRcB ? kRcB : 0) + tx; ll <= ii; ll += 16) {
            const int l = jn + ll;
            double v = M[i * ld + l];
#pragma unroll
            for (int u = 0; u < kRcB; ++u) v = fma(-li[u], M[l * ld + jb + u], v);
            M[i * ld + l] = v;
          }
        }
      }
    }
    __syncthreads();
  }
  if (bad && err) atomicExch(err, 1);
  RC_MARK(1);
  // ---- substitutions: one warp per right-hand side -------------------------
  for (int s0 = blockIdx.x * cpc; s0 < m; s0 += gridDim.x * cpc) {
    const int s = wid < cpc ? s0 + wid : m;
    double y[KPL];
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      y[c] = (s < m && i < kr) ? __ldg(beta + (int64_t)i * m + s) : 0.0;
    }
    // L y = b, block by block: z = W_b y_b, then the rows below
    for (int jb = 0; jb < K; jb += kRcB) {
      const int cs = jb >> 5, lb = jb & 31;
      const double own = rc_pick<KPL>(y, cs);
      const double* w = Wb + (jb / kRcB) * 64;
      double z[kRcB], x[kRcB];
#pragma unroll
      for (int t = 0; t < kRcB; ++t) z[t] = __shfl_sync(0xffffffffu, own, lb + t);
#pragma unroll
      for (int t = 0; t < kRcB; ++t) {
        double acc = 0.0;
#pragma unroll
        for (int u = 0; u <= t; ++u) acc = fma(w[t * kRcB + u], z[u], acc);
        x[t] = acc;
      }
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        const int i = lane + 32 * c;
        if (i >= jb && i < jb + kRcB) {
#pragma unroll
          for (int t = 0; t < kRcB; ++t)
            if (i == jb + t) y[c] = x[t];
        } else if (i >= jb + kRcB && i < K) {
          double v = y[c];
#pragma unroll
          for (int t = 0; t < kRcB; ++t) v = fma(-M[i * ld + jb + t], x[t], v);
          y[c] = v;
        }
      }
    }
    // L^T a = y, blocks from the last: x = W_b^T y_b, then the rows above
    for (int jb = K - kRcB; jb >= 0; jb -= kRcB) {
      const int cs = jb >> 5, lb = jb & 31;
      const double own = rc_pick<KPL>(y, cs);
      const double* w = Wb + (jb / kRcB) * 64;
      double z[kRcB], x[kRcB];
#pragma unroll
      for (int t = 0; t < kRcB; ++t) z[t] = __shfl_sync(0xffffffffu, own, lb + t);
#pragma unroll
      for (int t = 0; t < kRcB; ++t) {
        double acc = 0.0;
#pragma unroll
        for (int u = t; u < kRcB; ++u) acc = fma(w[u * kRcB + t], z[u], acc);
        x[t] = acc;
      }
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        const int i = lane + 32 * c;
        if (i >= jb && i < jb + kRcB) {
#pragma unroll
          for (int t = 0; t < kRcB; ++t)
            if (i == jb + t) y[c] = x[t];
        } else if (i < jb) {
          double v = y[c];
#pragma unroll
          for (int t = 0; t < kRcB; ++t) v = fma(-M[(jb + t) * ld + i], x[t], v);
          y[c] = v;
        }
      }
    }
    double* Yw = Y + (size_t)wid * K;
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      if (i < K) {
        const double v = (s < m && i < kr) ? y[c] : 0.0;
        Yw[i] = v;
        if (s < m && i < kr) {
          A64[(int64_t)i * m + s] = v;
          A32[(int64_t)i * m + s] = (float)v;
          if (AT32) AT32[(int64_t)s * ldt + i] = (float)v;     // codes transposed (eta x kp) for bbar
        }
      }
    }
  }
  RC_MARK(2);
  if (cpart) {
    __syncthreads();
    double* out = cpart + (size_t)blockIdx.x * kr * kr;
    for (int e = tid; e < kr * kr; e += kRcThreads) {
      const int a = e / kr, b = e % kr;
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) acc = fma(Y[w * K + a], Y[w * K + b], acc);
      out[e] = acc;
    }
  }
  __syncthreads();
  RC_MARK(3);
#undef RC_MARK
}

__global__ void k_cbar_finalize(const double* __restrict__ cpart, int nparts, int k, int eta,
                                const double* __restrict__ w_dev, double* __restrict__ C64,
                                float* __restrict__ C32) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const double keepd = w_dev[kCoefKeep], gc = w_dev[kCoefGainC];
  double s = 0.0;
  for (int b = 0; b < nparts; ++b) s += cpart[(size_t)b * k * k + e];
  const double c = keepd * C64[e] + (gc / eta) * s;
  C64[e] = c;
  C32[e] = (float)c;
}

}  // namespace somf
