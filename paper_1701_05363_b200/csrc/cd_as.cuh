// cd_as.cuh -- (a2) lasso / elastic-net / non-negative codes (Eq. somf_alpha,
// P:592-596) by cyclic coordinate descent WITH SUPPORT JUMPS (the survey's
// recommended K4 design, SURVEY §8c "Code-solve latency"):
//
//   minimise 1/2 a^T G a - beta^T a + l1 |a|_1 + l2/2 |a|^2  (a >= 0 if positive)
//
// The solution is unique (G + l2 I > 0 on the support), so any
// convergent path gives the oracle's value (reading R14).  Plain cyclic CD
// (k_cd) needs ~90 sweeps of k dependent coordinate steps at cfgB (k = 256);
// here, after a few warm sweeps, every CD sweep is followed by a JUMP: with S
// the current support and s its signs, solve the stationarity system of the
// face exactly,
//   (G_SS + l2 I) a_S = beta_S - l1 s_S                         (KKT on S)
// by a warp Cholesky in fp64, and accept a_S if its signs agree with s (then
// it is the minimiser over the orthant face containing the current point,
// so the objective does not increase).  The next CD sweep either confirms
// optimality (max |delta| <= tol, every off-support KKT condition holds) or
// moves the support; convergence is CD's.  Supports larger than kAsMax skip
// the jump (plain CD).  One warp per column, 4 warps per CTA; per warp the
// face system (kAsMax^2 doubles) lives in shared memory next to the packed
// fp32 Gram (k = 256 fits).
#pragma once
#include "common.cuh"
#include "solve.cuh"

namespace somf {

constexpr int kAsThreads = 128;     // 4 warps = 4 columns per CTA
constexpr int kAsMax = 48;          // largest support solved exactly
constexpr int kAsWarm = 6;          // CD sweeps before the first jump

// per-warp scratch: kAsMax x kAsMax doubles (A, then L) + kAsMax doubles (y) + kAsMax ints
__host__ __device__ constexpr size_t cd_as_warp_bytes() {
  return (size_t)kAsMax * kAsMax * 8 + (size_t)kAsMax * 8 + (size_t)kAsMax * 4;
}

// GT: the packed Gram's type in shared memory (double when it fits, else float)
template <int KPL, typename GT>
__global__ void __launch_bounds__(kAsThreads)
k_cd_as(const double* __restrict__ G, const double* __restrict__ beta, int k, int m,
        double l1, double l2, int positive, double tol, int max_sweeps,
        double* __restrict__ A64, float* __restrict__ A32, int* __restrict__ sweeps_out,
        float* __restrict__ AT32, int ldt, int64_t gstride) {
  // the B-bar kernel may launch now (programmatic dependent launch); it reads
  // the codes only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  // gstride > 0: a Gram per column (estimator (b)); one column (warp) per CTA
  G += (int64_t)blockIdx.x * gstride;
  extern __shared__ __align__(16) uint8_t as_smem[];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int np = k * (k + 1) / 2;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  uint8_t* wbase = as_smem + (size_t)wid * cd_as_warp_bytes();
  double* Af = reinterpret_cast<double*>(wbase);                  // kAsMax x kAsMax
  double* yv = Af + kAsMax * kAsMax;                              // kAsMax
  int* sidx = reinterpret_cast<int*>(yv + kAsMax);                // kAsMax
  GT* Pk = reinterpret_cast<GT*>(as_smem + (size_t)nw * cd_as_warp_bytes());   // packed upper triangle
  for (int e = tid; e < np; e += nt) {
    int lo = 0, hi = k - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (packed_off(mid, k) <= e) lo = mid; else hi = mid - 1;
    }
    const int i = lo, j = i + (e - packed_off(i, k));
    Pk[e] = (GT)G[(int64_t)i * k + j];
  }
  __syncthreads();
  for (int s = blockIdx.x * nw + wid; s < m; s += gridDim.x * nw) {
    double alpha[KPL], g[KPL], den[KPL], rden[KPL], b[KPL];
    int roff[KPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int row = lane + 32 * i;
      alpha[i] = 0.0;
      b[i] = row < k ? beta[(int64_t)row * m + s] : 0.0;
      g[i] = b[i];
      den[i] = row < k ? (double)packed_get(Pk, row, row, k) + l2 : 1.0;
      rden[i] = den[i] > 0.0 ? 1.0 / den[i] : 0.0;
      roff[i] = packed_off(row < k ? row : 0, k);
    }
    int sweep = 0;
    for (; sweep < max_sweeps; ++sweep) {
      // ---- one cyclic CD sweep (as k_cd) ----
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
            if (!(den[slot] > 0.0)) nv = 0.0;                          // R12
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
      if (sweep + 1 < kAsWarm) continue;
      // ---- jump: exact solve on the current support ----
      int n = 0;
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        const unsigned msk = __ballot_sync(0xffffffffu, alpha[slot] != 0.0);
        const int pos = n + __popc(msk & ((1u << lane) - 1u));
        if (alpha[slot] != 0.0 && pos < kAsMax) sidx[pos] = slot * 32 + lane;
        n += __popc(msk);
      }
      if (n == 0 || n > kAsMax) continue;
      __syncwarp();
      // A = G_SS + l2 I (lower triangle), y = beta_S - l1 sign_S
      for (int e = lane; e < n * n; e += 32) {
        const int r = e / n, c = e % n;
        if (c <= r) {
          const int jr = sidx[r], jc = sidx[c];
          Af[r * kAsMax + c] = (double)packed_get(Pk, jr, jc, k) + (r == c ? l2 : 0.0);
        }
      }
      for (int r = lane; r < n; r += 32) yv[r] = 0.0;
      __syncwarp();
      // beta_S and signs: the owner lane of coordinate j writes y
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        if (alpha[slot] != 0.0) {
          // position of coordinate (slot, lane) in sidx: recount (cheap, n <= 48)
          const int j = slot * 32 + lane;
          for (int r = 0; r < n; ++r)
            if (sidx[r] == j) yv[r] = b[slot] - l1 * (alpha[slot] > 0.0 ? 1.0 : -1.0);
        }
      }
      __syncwarp();
      // Cholesky (right-looking, column by column; rows by lane)
      bool ok = true;
      for (int c = 0; c < n; ++c) {
        const double d = Af[c * kAsMax + c];
        if (!(d > 0.0)) { ok = false; break; }
        const double ld = sqrt(d), il = 1.0 / ld;
        __syncwarp();
        for (int r = c + 1 + lane; r < n; r += 32) Af[r * kAsMax + c] *= il;
        __syncwarp();
        if (lane == 0) Af[c * kAsMax + c] = ld;
        for (int r = c + 1 + lane; r < n; r += 32) {
          const double lrc = Af[r * kAsMax + c];
          for (int q = c + 1; q <= r; ++q) Af[r * kAsMax + q] = fma(-lrc, Af[q * kAsMax + c], Af[r * kAsMax + q]);
        }
        __syncwarp();
      }
      ok = __all_sync(0xffffffffu, ok);
      if (!ok) continue;
      // L z = y (column-oriented), then L^T x = z
      for (int c = 0; c < n; ++c) {
        const double zc = yv[c] / Af[c * kAsMax + c];
        __syncwarp();
        if (lane == 0) yv[c] = zc;
        for (int r = c + 1 + lane; r < n; r += 32) yv[r] = fma(-Af[r * kAsMax + c], zc, yv[r]);
        __syncwarp();
      }
      for (int c = n - 1; c >= 0; --c) {
        double acc = 0.0;
        for (int r = c + 1 + lane; r < n; r += 32) acc = fma(Af[r * kAsMax + c], yv[r], acc);
        acc = warp_sum(acc);
        const double xc = (yv[c] - acc) / Af[c * kAsMax + c];
        __syncwarp();
        if (lane == 0) yv[c] = xc;
        __syncwarp();
      }
      // accept only if every sign agrees (then the face minimiser is feasible)
      bool agree = true;
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        if (alpha[slot] != 0.0) {
          const int j = slot * 32 + lane;
          for (int r = 0; r < n; ++r)
            if (sidx[r] == j) agree &= (alpha[slot] > 0.0) ? (yv[r] > 0.0) : (yv[r] < 0.0);
        }
      }
      agree = __all_sync(0xffffffffu, agree);
      if (!agree) continue;
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        if (alpha[slot] != 0.0) {
          const int j = slot * 32 + lane;
          for (int r = 0; r < n; ++r)
            if (sidx[r] == j) alpha[slot] = yv[r];
        }
      }
      // g = beta - G alpha (alpha supported on S)
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int row = lane + 32 * i;
        double acc = 0.0;
        if (row < k) {
          for (int r = 0; r < n; ++r) acc = fma((double)packed_get(Pk, row, sidx[r], k), yv[r], acc);
        }
        g[i] = b[i] - acc;
      }
      __syncwarp();
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

}  // namespace somf
