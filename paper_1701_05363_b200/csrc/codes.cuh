// codes.cuh -- (a2) ridge codes and (a3) Cbar, v2:
//
//  k_ridge_codes<KPL> : alpha = (G + lambda I)^-1 beta  (Eq. somf_alpha,
//                  P:592-596, nu = 1, no positivity), k <= 32 KPL.
//                  Every CTA factorises G + lambda I redundantly in shared
//                  memory (fp64 LL^T, right-looking in 8-column panels: the
//                  8 x 8 diagonal block is factorised in every thread's
//                  registers, the panel rows below are solved one row per
//                  thread, then one rank-4 trailing update over a 16 x 16
//                  thread grid: 2 barriers per 4 columns).  Then each warp
//                  solves one right-hand side with 4-row block substitutions
//                  (the solution in registers, lane l holding rows l, l+32,
//                  ...; one shuffle round per 4 rows).  Each CTA also writes
//                  its partial sum_s alpha_s alpha_s^T for the Cbar update.
//  k_cbar_finalize : Cbar <- (1 - w) Cbar + (w / eta) sum_b partial_b
//                  (Eq. somf_partial, batch mean R4), partials added in
//                  block order (deterministic).
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kRcThreads = 256;
constexpr int kRcMaxK = 160;
constexpr int kRcPW = 4;          // panel width of the factorisation (8 measured slower)
constexpr int kRcSB = 8;          // block height of the substitutions (8 measured faster than 4); multiple of kRcPW
constexpr int kRcInvKPL = 0;      // k <= 32 kRcInvKPL: explicit-inverse solve (measured slower on B200 for k = 70: off)

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

// smem: k x (k+1) doubles (L, 1/L_jj on the diagonal) + 8 warps x k doubles
template <int KPL>
__global__ void __launch_bounds__(kRcThreads)
k_ridge_codes(const double* __restrict__ G, const double* __restrict__ beta, int k, int m, double lam,
              double* __restrict__ A64, float* __restrict__ A32, float* __restrict__ AT32, int ldt,
              double* __restrict__ cpart, int* __restrict__ err, long long* __restrict__ prof) {
  // the B-bar kernel may launch now (programmatic dependent launch); it reads
  // the codes only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
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
  // the factorisation and the solves run on K4 = k rounded up to 4 (identity
  // padding, zero right-hand sides): every 4-column panel / 4-row block is
  // full, so the loops are branch-free and the loads can be hoisted
  const int kr = k;
  k = (k + kRcSB - 1) & ~(kRcSB - 1);
  const int ld = k + 1;
  double* M = rc_smem;                              // k x ld, lower triangle
  double* Y = rc_smem + (size_t)k * ld;             // 8 x k
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ty = tid >> 4, tx = tid & 15;
#pragma unroll 4
  for (int e = tid; e < k * k; e += kRcThreads) {
    const int i = e / k, j = e % k;
    const double g = (i < kr && j < kr) ? G[(int64_t)i * kr + j] + (i == j ? lam : 0.0) : (i == j ? 1.0 : 0.0);
    if (j <= i) M[i * ld + j] = g;
  }
  __syncthreads();
  RC_MARK(0);
  bool bad = false;
  for (int p0 = 0; p0 < k; p0 += kRcPW) {
    constexpr int pb = kRcPW;
    // 4 x 4 diagonal block, factorised in registers by every thread
    double Ld[kRcPW][kRcPW];
#pragma unroll
    for (int a = 0; a < kRcPW; ++a)
#pragma unroll
      for (int c = 0; c < kRcPW; ++c) Ld[a][c] = (a < pb && c <= a) ? M[(p0 + a) * ld + p0 + c] : 0.0;
    double inv[kRcPW];
#pragma unroll
    for (int c = 0; c < kRcPW; ++c) {
      if (c < pb) {
        double d = Ld[c][c];
#pragma unroll
        for (int u = 0; u < kRcPW; ++u)
          if (u < c) d -= Ld[c][u] * Ld[c][u];
        bad |= !(d > 0.0);
        const double ir = d > 0.0 ? rc_rsqrt(d) : 0.0;
        inv[c] = ir;
        Ld[c][c] = d * ir;
#pragma unroll
        for (int a = 0; a < kRcPW; ++a) {
          if (a > c && a < pb) {
            double v = Ld[a][c];
#pragma unroll
            for (int u = 0; u < kRcPW; ++u)
              if (u < c) v -= Ld[a][u] * Ld[c][u];
            Ld[a][c] = v * inv[c];
          }
        }
      } else {
        inv[c] = 0.0;
      }
    }
    // panel rows below: L[i][p0..p0+pb) = M[i][p0..] L_D^-T  (one row per thread)
    for (int i = p0 + pb + tid; i < k; i += kRcThreads) {
      double x[kRcPW];
#pragma unroll
      for (int c = 0; c < kRcPW; ++c) {
        if (c < pb) {
          double v = M[i * ld + p0 + c];
#pragma unroll
          for (int u = 0; u < kRcPW; ++u)
            if (u < c) v -= x[u] * Ld[c][u];
          x[c] = v * inv[c];
        } else {
          x[c] = 0.0;
        }
      }
#pragma unroll
      for (int c = 0; c < kRcPW; ++c)
        if (c < pb) M[i * ld + p0 + c] = x[c];
    }
    __syncthreads();                                // panel reads of the block done
    // (static register indices only: a dynamic index would put Ld in local memory)
#pragma unroll
    for (int a = 0; a < kRcPW; ++a)
#pragma unroll
      for (int c = 0; c < kRcPW; ++c)
        if (tid == kRcPW * a + c && a < pb && c <= a) M[(p0 + a) * ld + p0 + c] = (a == c) ? inv[a] : Ld[a][c];
    // rank-4 trailing update: M[i][l] -= sum_c L[i][p0+c] L[l][p0+c], p0+pb <= l <= i.
    // Thread (ty, tx) owns rows r0+ty+16a and columns r0+tx+16b; the panel
    // values of its columns are loaded once into registers (NS = KMAX/16 slots).
    {
      constexpr int NS = (32 * KPL + 15) / 16;
      const int r0 = p0 + pb, n = k - r0;
      double lj[NS][kRcPW];
#pragma unroll
      for (int bb = 0; bb < NS; ++bb) {
        const int ll = tx + 16 * bb;
#pragma unroll
        for (int c = 0; c < kRcPW; ++c) lj[bb][c] = (ll < n && c < pb) ? M[(r0 + ll) * ld + p0 + c] : 0.0;
      }
      for (int ii = ty; ii < n; ii += 16) {
        const int i = r0 + ii;
        double li[kRcPW];
#pragma unroll
        for (int c = 0; c < kRcPW; ++c) li[c] = c < pb ? M[i * ld + p0 + c] : 0.0;
#pragma unroll
        for (int bb = 0; bb < NS; ++bb) {
          const int ll = tx + 16 * bb;
          if (ll <= ii) {
            double* mp = M + i * ld + r0 + ll;
            double v = *mp;
#pragma unroll
            for (int c = 0; c < kRcPW; ++c) v -= li[c] * lj[bb][c];
            *mp = v;
          }
        }
      }
    }
    __syncthreads();
  }
  if (bad && err) atomicExch(err, 1);
  RC_MARK(1);

  if constexpr (KPL <= kRcInvKPL) {
    // ---- explicit inverse W = L^-1 (column j by thread j), then alpha = W^T (W beta):
    // two triangular mat-vecs per right-hand side, no serial substitution chain
    double* W = Y + (size_t)8 * k;                    // k x ld, lower triangle
    for (int j = tid; j < k; j += kRcThreads) {
      W[j * ld + j] = M[j * ld + j];
      for (int i = j + 1; i < k; ++i) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int l = j;
        for (; l + 3 < i; l += 4) {
          a0 = fma(M[i * ld + l], W[l * ld + j], a0);
          a1 = fma(M[i * ld + l + 1], W[(l + 1) * ld + j], a1);
          a2 = fma(M[i * ld + l + 2], W[(l + 2) * ld + j], a2);
          a3 = fma(M[i * ld + l + 3], W[(l + 3) * ld + j], a3);
        }
        for (; l < i; ++l) a0 = fma(M[i * ld + l], W[l * ld + j], a0);
        W[i * ld + j] = -M[i * ld + i] * ((a0 + a1) + (a2 + a3));
      }
    }
    __syncthreads();
    RC_MARK(7);       // prof slot 79: the inverse
    double* Yw = Y + (size_t)wid * k;
    for (int s0 = blockIdx.x * 8; s0 < m; s0 += gridDim.x * 8) {
      const int s = s0 + wid;
      for (int i = lane; i < k; i += 32) Yw[i] = (s < m && i < kr) ? beta[(int64_t)i * m + s] : 0.0;
      __syncwarp();
      double y[KPL];
#pragma unroll
      for (int c = 0; c < KPL; ++c) {                 // y = W beta (rows i >= l)
        const int i = lane + 32 * c;
        double a0 = 0.0, a1 = 0.0;
        if (i < k) {
          int l = 0;
          for (; l + 1 <= i; l += 2) {
            a0 = fma(W[i * ld + l], Yw[l], a0);
            a1 = fma(W[i * ld + l + 1], Yw[l + 1], a1);
          }
          if (l <= i) a0 = fma(W[i * ld + l], Yw[l], a0);
        }
        y[c] = a0 + a1;
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        const int i = lane + 32 * c;
        if (i < k) Yw[i] = y[c];
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < KPL; ++c) {                 // alpha = W^T y (rows l >= i)
        const int i = lane + 32 * c;
        double a0 = 0.0, a1 = 0.0;
        if (i < k) {
          int l = i;
          for (; l + 1 < k; l += 2) {
            a0 = fma(W[l * ld + i], Yw[l], a0);
            a1 = fma(W[(l + 1) * ld + i], Yw[l + 1], a1);
          }
          if (l < k) a0 = fma(W[l * ld + i], Yw[l], a0);
        }
        y[c] = a0 + a1;
      }
      __syncwarp();
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        const int i = lane + 32 * c;
        if (i < k) {
          const double v = s < m ? y[c] : 0.0;
          Yw[i] = v;
          if (s < m && i < kr) {
            A64[(int64_t)i * m + s] = v;
            A32[(int64_t)i * m + s] = (float)v;
            if (AT32) AT32[(int64_t)s * ldt + i] = (float)v;
          }
        }
      }
      __syncwarp();
    }
  } else {
  // ---- substitutions: one warp per right-hand side, 4 rows per shuffle round ----
  for (int s0 = blockIdx.x * 8; s0 < m; s0 += gridDim.x * 8) {
    const int s = s0 + wid;
    double y[KPL];
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      y[c] = (s < m && i < kr) ? beta[(int64_t)i * m + s] : 0.0;
    }
    // L y = b
    for (int jb = 0; jb < k; jb += kRcSB) {
      constexpr int pb = kRcSB;
      const int cs = jb >> 5, lb = jb & 31;
      const double own = rc_pick<KPL>(y, cs);
      double z[kRcSB];
#pragma unroll
      for (int t = 0; t < kRcSB; ++t) z[t] = __shfl_sync(0xffffffffu, own, lb + t);
#pragma unroll
      for (int t = 0; t < kRcSB; ++t) {
        if (t < pb) {
          double v = z[t];
#pragma unroll
          for (int u = 0; u < kRcSB; ++u)
            if (u < t) v -= M[(jb + t) * ld + jb + u] * z[u];
          z[t] = v * M[(jb + t) * ld + jb + t];
        }
      }
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        const int i = lane + 32 * c;
        if (i >= jb && i < jb + pb) {
#pragma unroll
          for (int t = 0; t < kRcSB; ++t)
            if (i == jb + t) y[c] = z[t];
        } else if (i >= jb + pb && i < k) {
          double v = y[c];
#pragma unroll
          for (int t = 0; t < kRcSB; ++t)
            if (t < pb) v -= M[i * ld + jb + t] * z[t];
          y[c] = v;
        }
      }
    }
    // L^T x = y
    for (int jb = ((k - 1) / kRcSB) * kRcSB; jb >= 0; jb -= kRcSB) {
      constexpr int pb = kRcSB;
      const int cs = jb >> 5, lb = jb & 31;
      const double own = rc_pick<KPL>(y, cs);
      double z[kRcSB];
#pragma unroll
      for (int t = 0; t < kRcSB; ++t) z[t] = __shfl_sync(0xffffffffu, own, lb + t);
#pragma unroll
      for (int t = kRcSB - 1; t >= 0; --t) {
        if (t < pb) {
          double v = z[t];
#pragma unroll
          for (int u = 0; u < kRcSB; ++u)
            if (u > t && u < pb) v -= M[(jb + u) * ld + jb + t] * z[u];
          z[t] = v * M[(jb + t) * ld + jb + t];
        }
      }
#pragma unroll
      for (int c = 0; c < KPL; ++c) {
        const int i = lane + 32 * c;
        if (i >= jb && i < jb + pb) {
#pragma unroll
          for (int t = 0; t < kRcSB; ++t)
            if (i == jb + t) y[c] = z[t];
        } else if (i < jb) {
          double v = y[c];
#pragma unroll
          for (int t = 0; t < kRcSB; ++t)
            if (t < pb) v -= M[(jb + t) * ld + i] * z[t];
          y[c] = v;
        }
      }
    }
    double* Yw = Y + (size_t)wid * k;
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      if (i < k) {
        const double v = s < m ? y[c] : 0.0;
        Yw[i] = v;
        if (s < m && i < kr) {
          A64[(int64_t)i * m + s] = v;
          A32[(int64_t)i * m + s] = (float)v;
          if (AT32) AT32[(int64_t)s * ldt + i] = (float)v;     // codes transposed (eta x kp) for bbar
        }
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
      for (int w = 0; w < 8; ++w) acc += Y[w * k + a] * Y[w * k + b];
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
  const double w = *w_dev;
  double s = 0.0;
  for (int b = 0; b < nparts; ++b) s += cpart[(size_t)b * k * k + e];
  const double c = (1.0 - w) * C64[e] + (w / eta) * s;
  C64[e] = c;
  C32[e] = (float)c;
}

}  // namespace somf
