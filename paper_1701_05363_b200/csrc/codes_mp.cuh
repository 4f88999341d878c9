// codes_mp.cuh -- (a2) ridge codes alpha = (G + lambda I)^-1 beta (Eq. somf_alpha,
// P:592-596, nu = 1, no positivity) in MIXED precision: the Cholesky factor
// and the triangular substitutions in fp32 (half the latency of every link of
// the factorisation chain: FFMA vs DFMA, MUFU rsqrt), then one step of
// iterative refinement with the residual in fp64:
//   alpha0 = L^-T L^-1 beta (fp32),  r = beta - (G + lambda I) alpha0 (fp64),
//   alpha = alpha0 + L^-T L^-1 r.
// With eps32 ~ 6e-8 and the conditioning of G + lambda I at the configs
// (lambda = 1e-3, unit-norm atoms: kappa <~ 1e3-1e4) the refined alpha is at
// the fp64 solve to ~(kappa k eps32)^2, far inside the 1e-4 parity bar
// (DESIGN.md §5).  Same CTA structure as k_ridge_codes: every CTA factorises
// redundantly (4-column panels, register-resident diagonal block), one warp
// per right-hand side, 8 right-hand sides per CTA, partial sum_s alpha_s
// alpha_s^T per CTA for the Cbar update.
#pragma once
#include "common.cuh"
#include "codes.cuh"

namespace somf {

template <int KPL>
__device__ __forceinline__ float rcf_pick(const float (&y)[KPL], int c) {
  float v = 0.f;
#pragma unroll
  for (int i = 0; i < KPL; ++i)
    if (i == c) v = y[i];
  return v;
}

// L y = b then L^T x = y for one right-hand side held by a warp (lane l holds
// rows l, l + 32, ...); M: k x ld lower triangle with 1/L_jj on the diagonal
template <int KPL>
__device__ __forceinline__ void rcf_subst(float (&y)[KPL], const float* M, int ld, int k, int lane) {
  for (int jb = 0; jb < k; jb += kRcSB) {
    const int cs = jb >> 5, lb = jb & 31;
    const float own = rcf_pick<KPL>(y, cs);
    float z[kRcSB];
#pragma unroll
    for (int t = 0; t < kRcSB; ++t) z[t] = __shfl_sync(0xffffffffu, own, lb + t);
#pragma unroll
    for (int t = 0; t < kRcSB; ++t) {
      float v = z[t];
#pragma unroll
      for (int u = 0; u < kRcSB; ++u)
        if (u < t) v = fmaf(-M[(jb + t) * ld + jb + u], z[u], v);
      z[t] = v * M[(jb + t) * ld + jb + t];
    }
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      if (i >= jb && i < jb + kRcSB) {
#pragma unroll
        for (int t = 0; t < kRcSB; ++t)
          if (i == jb + t) y[c] = z[t];
      } else if (i >= jb + kRcSB && i < k) {
        float v = y[c];
#pragma unroll
        for (int t = 0; t < kRcSB; ++t) v = fmaf(-M[i * ld + jb + t], z[t], v);
        y[c] = v;
      }
    }
  }
  for (int jb = ((k - 1) / kRcSB) * kRcSB; jb >= 0; jb -= kRcSB) {
    const int cs = jb >> 5, lb = jb & 31;
    const float own = rcf_pick<KPL>(y, cs);
    float z[kRcSB];
#pragma unroll
    for (int t = 0; t < kRcSB; ++t) z[t] = __shfl_sync(0xffffffffu, own, lb + t);
#pragma unroll
    for (int t = kRcSB - 1; t >= 0; --t) {
      float v = z[t];
#pragma unroll
      for (int u = 0; u < kRcSB; ++u)
        if (u > t) v = fmaf(-M[(jb + u) * ld + jb + t], z[u], v);
      z[t] = v * M[(jb + t) * ld + jb + t];
    }
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      if (i >= jb && i < jb + kRcSB) {
#pragma unroll
        for (int t = 0; t < kRcSB; ++t)
          if (i == jb + t) y[c] = z[t];
      } else if (i < jb) {
        float v = y[c];
#pragma unroll
        for (int t = 0; t < kRcSB; ++t) v = fmaf(-M[(jb + t) * ld + i], z[t], v);
        y[c] = v;
      }
    }
  }
}

// smem: 8 warps x k4 doubles (alpha of each warp's column) + k4 x kr doubles
// (G + lambda I for the residual) + k4 x (k4 + 1) floats (L)
template <int KPL, int PW>
__global__ void __launch_bounds__(kRcThreads)
k_ridge_mp(const double* __restrict__ G, const double* __restrict__ beta, int k, int m, double lam,
           double* __restrict__ A64, float* __restrict__ A32, float* __restrict__ AT32, int ldt,
           double* __restrict__ cpart, int* __restrict__ err, long long* __restrict__ prof) {
  // the B-bar kernel may launch now (programmatic dependent launch); it reads
  // the codes only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ double rcm_smem[];
  long long t_mark = clock64();
#define RCM_MARK(slot)                                                    \
  do {                                                                    \
    if (prof && blockIdx.x == 0 && threadIdx.x == 0) {                    \
      const long long now_ = clock64();                                   \
      prof[slot] += now_ - t_mark;                                        \
      t_mark = now_;                                                      \
    }                                                                     \
  } while (0)
  const int kr = k;
  k = (k + kRcSB - 1) & ~(kRcSB - 1);                 // identity padding to a multiple of 8
  const int ld = k + 1;
  double* Y = rcm_smem;                               // 8 x k doubles
  double* Gs = Y + (size_t)8 * k;                     // kr x (kr + 1) doubles: G + lambda I
  const int ldg = kr + 1;
  float* M = reinterpret_cast<float*>(Gs + (size_t)kr * ldg);   // k x ld, lower triangle
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ty = tid >> 4, tx = tid & 15;
#pragma unroll 4
  for (int e = tid; e < k * k; e += kRcThreads) {
    const int i = e / k, j = e % k;
    const double g = (i < kr && j < kr) ? G[(int64_t)i * kr + j] + (i == j ? lam : 0.0) : (i == j ? 1.0 : 0.0);
    if (j <= i) M[i * ld + j] = (float)g;
    if (i < kr && j < kr) Gs[i * ldg + j] = g;
  }
  __syncthreads();
  RCM_MARK(0);
  bool bad = false;
  for (int p0 = 0; p0 < k; p0 += PW) {
    // 4 x 4 diagonal block, factorised in registers by every thread
    float Ld[PW][PW];
#pragma unroll
    for (int a = 0; a < PW; ++a)
#pragma unroll
      for (int c = 0; c < PW; ++c) Ld[a][c] = c <= a ? M[(p0 + a) * ld + p0 + c] : 0.f;
    float inv[PW];
#pragma unroll
    for (int c = 0; c < PW; ++c) {
      float d = Ld[c][c];
#pragma unroll
      for (int u = 0; u < PW; ++u)
        if (u < c) d = fmaf(-Ld[c][u], Ld[c][u], d);
      bad |= !(d > 0.f);
      float ir = d > 0.f ? rsqrtf(d) : 0.f;
      ir = ir * fmaf(-0.5f * d, ir * ir, 1.5f);      // one Newton step: rel. error ~1e-7
      inv[c] = ir;
      Ld[c][c] = d * ir;
#pragma unroll
      for (int a = 0; a < PW; ++a) {
        if (a > c) {
          float v = Ld[a][c];
#pragma unroll
          for (int u = 0; u < PW; ++u)
            if (u < c) v = fmaf(-Ld[a][u], Ld[c][u], v);
          Ld[a][c] = v * inv[c];
        }
      }
    }
    // panel rows below: one row per thread
    for (int i = p0 + PW + tid; i < k; i += kRcThreads) {
      float x[PW];
#pragma unroll
      for (int c = 0; c < PW; ++c) {
        float v = M[i * ld + p0 + c];
#pragma unroll
        for (int u = 0; u < PW; ++u)
          if (u < c) v = fmaf(-x[u], Ld[c][u], v);
        x[c] = v * inv[c];
      }
#pragma unroll
      for (int c = 0; c < PW; ++c) M[i * ld + p0 + c] = x[c];
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < PW; ++a)
#pragma unroll
      for (int c = 0; c < PW; ++c)
        if (tid == PW * a + c && c <= a) M[(p0 + a) * ld + p0 + c] = (a == c) ? inv[a] : Ld[a][c];
    // rank-4 trailing update over a 16 x 16 thread grid
    {
      constexpr int NS = (32 * KPL + 15) / 16;
      const int r0 = p0 + PW, n = k - r0;
      float lj[NS][PW];
#pragma unroll
      for (int bb = 0; bb < NS; ++bb) {
        const int ll = tx + 16 * bb;
#pragma unroll
        for (int c = 0; c < PW; ++c) lj[bb][c] = ll < n ? M[(r0 + ll) * ld + p0 + c] : 0.f;
      }
      for (int ii = ty; ii < n; ii += 16) {
        const int i = r0 + ii;
        float li[PW];
#pragma unroll
        for (int c = 0; c < PW; ++c) li[c] = M[i * ld + p0 + c];
#pragma unroll
        for (int bb = 0; bb < NS; ++bb) {
          const int ll = tx + 16 * bb;
          if (ll <= ii) {
            float* mp = M + i * ld + r0 + ll;
            float v = *mp;
#pragma unroll
            for (int c = 0; c < PW; ++c) v = fmaf(-li[c], lj[bb][c], v);
            *mp = v;
          }
        }
      }
    }
    __syncthreads();
  }
  if (bad && err) atomicExch(err, 1);
  RCM_MARK(1);
  // ---- solve + one refinement step, one warp per right-hand side ----
  double* Yw = Y + (size_t)wid * k;
  for (int s0 = blockIdx.x * 8; s0 < m; s0 += gridDim.x * 8) {
    const int s = s0 + wid;
    double b64[KPL], al[KPL];
    float y[KPL];
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      b64[c] = (s < m && i < kr) ? beta[(int64_t)i * m + s] : 0.0;
      y[c] = (float)b64[c];
    }
    rcf_subst<KPL>(y, M, ld, k, lane);
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      al[c] = (double)y[c];
      if (i < k) Yw[i] = al[c];
    }
    __syncwarp();
    // r = beta - (G + lambda I) alpha0 in fp64 (G rows from L2)
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      double r = 0.0;
      if (i < kr) {
        const double* gi = Gs + (size_t)i * ldg;          // includes lambda on the diagonal
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int j = 0;
        for (; j + 3 < kr; j += 4) {
          a0 = fma(gi[j], Yw[j], a0);
          a1 = fma(gi[j + 1], Yw[j + 1], a1);
          a2 = fma(gi[j + 2], Yw[j + 2], a2);
          a3 = fma(gi[j + 3], Yw[j + 3], a3);
        }
        for (; j < kr; ++j) a0 = fma(gi[j], Yw[j], a0);
        r = b64[c] - ((a0 + a1) + (a2 + a3));
      }
      y[c] = (float)r;
    }
    __syncwarp();
    rcf_subst<KPL>(y, M, ld, k, lane);
#pragma unroll
    for (int c = 0; c < KPL; ++c) {
      const int i = lane + 32 * c;
      if (i < k) {
        const double v = (s < m && i < kr) ? al[c] + (double)y[c] : 0.0;
        Yw[i] = v;
        if (s < m && i < kr) {
          A64[(int64_t)i * m + s] = v;
          A32[(int64_t)i * m + s] = (float)v;
          if (AT32) AT32[(int64_t)s * ldt + i] = (float)v;     // codes transposed (eta x kp) for bbar
        }
      }
    }
    __syncwarp();
  }
  RCM_MARK(2);
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
  RCM_MARK(3);
#undef RCM_MARK
}

}  // namespace somf
