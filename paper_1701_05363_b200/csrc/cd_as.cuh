// cd_as.cuh -- (a2) lasso / elastic-net / non-negative codes (Eq. somf_alpha,
// P:592-596) by cyclic coordinate descent WITH SUPPORT JUMPS (the survey's
// recommended K4 design, SURVEY §8c "Code-solve latency"):
//
//   minimise 1/2 a^T G a - beta^T a + l1 |a|_1 + l2/2 |a|^2  (a >= 0 if positive)
//
// The solution is unique (G + l2 I > 0 on the support), so any
// convergent path gives the oracle's value (readings R14, R14b).  Plain cyclic
// CD (k_cd) needs ~90 sweeps of k dependent coordinate steps at cfgB (k = 256)
// and ~700 at cfgD (nonneg ridge on an NMF Gram, cond ~5e3); here:
//
//  * each CD sweep is exact cyclic CD, but the coordinates whose update is
//    zero (most of them: the codes are sparse) cost nothing: all 32 lanes of a
//    slot compute their candidate update from the current gradient, a ballot
//    finds the FIRST nonzero one in cyclic order, only that one is applied
//    (broadcast + gradient update), and the lanes after it recompute;
//  * after kAsWarm sweeps, a sweep that left the support unchanged (or the
//    kAsForce-th sweep without one) is followed by a JUMP towards the
//    minimiser of the current orthant face: with S the support and s its signs,
//    solve (G_SS + l2 I) y = beta_S - l1 s_S (warp Cholesky, fp64).  If every
//    sign of y agrees, a_S <- y.  Otherwise move a_S along the segment towards
//    y up to the first coordinate that reaches zero, drop it, and solve again
//    on the smaller face (the feature-sign / active-set line search: the
//    objective is convex on the face, so it never increases).  The next CD
//    sweep confirms optimality (max |delta| <= tol) or moves the support.
//
// One warp per column; `nw` warps per CTA share the packed Gram in shared
// memory (fp64 when it fits, else fp32); each warp has a face scratch for
// supports up to `nmax` coordinates (larger supports skip the jump: plain CD).
#pragma once
#include "common.cuh"
#include "solve.cuh"

namespace somf {

constexpr int kAsWarm = 3;          // CD sweeps before the first jump
constexpr int kAsForce = 4;         // sweeps without a jump after which one is tried anyway
constexpr int kAsMaxLs = 3;         // face solves per jump (the line search's re-solves included)
constexpr int kAsRowsPerLane = 4;   // face rows per lane in the factorisation (nmax <= 128)

// per-warp scratch: packed lower face matrix, y, a_S, sidx, and a dense k-vector
__host__ __device__ constexpr size_t cd_as_warp_bytes(int nmax, int k) {
  return ((size_t)nmax * (nmax + 1) / 2 + 2 * (size_t)nmax + (size_t)((k + 1) & ~1)) * 8 +
         (size_t)((nmax + 3) & ~3) * 4;
}

__device__ __forceinline__ int pl_idx(int r, int c) { return (r * (r + 1) >> 1) + c; }   // packed lower, c <= r

// GT: the packed Gram's type in shared memory (double when it fits, else float)
template <int KPL, typename GT>
__global__ void __launch_bounds__(128)
k_cd_as(const double* __restrict__ G, const double* __restrict__ beta, int k, int m,
        double l1, double l2, int positive, double tol, int max_sweeps, int nmax,
        double* __restrict__ A64, float* __restrict__ A32, int* __restrict__ sweeps_out,
        float* __restrict__ AT32, int ldt, int64_t gstride, long long* __restrict__ prof) {
  // the B-bar kernel may launch now (programmatic dependent launch); it reads
  // the codes only after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  // gstride > 0: a Gram per column (estimator (b)); one column (warp) per CTA
  G += (int64_t)blockIdx.x * gstride;
  extern __shared__ __align__(16) uint8_t as_smem[];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int np = k * (k + 1) / 2;
  const int lane = tid & 31, wid = tid >> 5, nw = nt >> 5;
  const size_t wbytes = cd_as_warp_bytes(nmax, k);
  uint8_t* wbase = as_smem + (size_t)wid * wbytes;
  double* Af = reinterpret_cast<double*>(wbase);                  // nmax (nmax+1)/2, packed lower
  double* yv = Af + (size_t)nmax * (nmax + 1) / 2;                // nmax
  double* av = yv + nmax;                                         // nmax: a_S in sidx order
  double* anew = av + nmax;                                       // k: dense result of a jump
  int* sidx = reinterpret_cast<int*>(anew + ((k + 1) & ~1));      // nmax
  GT* Pk = reinterpret_cast<GT*>(as_smem + (size_t)nw * wbytes);  // packed upper triangle
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
    // diagnostics (prof != nullptr; somf_bcd_phase_cycles slots 84..91)
    long long c_sw = 0, c_jump = 0, n_solve = 0, n_sum = 0, n_agree = 0;
    int n_max = 0;
    long long t0 = prof ? clock64() : 0;
    // support of the previous sweep (one ballot per slot): a jump is tried once
    // the sweeps stop changing the support (the face solve then usually agrees
    // in sign at once), or after kAsForce sweeps without one
    unsigned smask[KPL];
#pragma unroll
    for (int i = 0; i < KPL; ++i) smask[i] = 0u;
    int since_jump = 0;
    for (; sweep < max_sweeps; ++sweep) {
      // ---- one cyclic CD sweep; zero updates skipped by ballot ----
      double maxd = 0.0;
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        const int jl = slot * 32 + lane;
        int ol = 0;
        while (ol < 32) {
          // candidate update of my coordinate from the current gradient
          double nv = 0.0, delta = 0.0;
          if (jl < k && lane >= ol) {
            const double gjj = den[slot] - l2;
            const double z = g[slot] + gjj * alpha[slot];
            if (!(den[slot] > 0.0)) nv = 0.0;                          // R12
            else if (positive) nv = fmax(z - l1, 0.0) * rden[slot];
            else nv = copysign(fmax(fabs(z) - l1, 0.0), z) * rden[slot];
            delta = nv - alpha[slot];
          }
          const unsigned bal = __ballot_sync(0xffffffffu, delta != 0.0);
          if (bal == 0u) break;
          const int o = __ffs(bal) - 1;                 // first nonzero update in cyclic order
          const double dl = __shfl_sync(0xffffffffu, delta, o);
          if (lane == o) alpha[slot] = nv;
          maxd = fmax(maxd, fabs(dl));
          const int j = slot * 32 + o;
          const int joff = packed_off(j, k);
#pragma unroll
          for (int i = 0; i < KPL; ++i) {
            const int row = lane + 32 * i;
            const int a = row <= j ? roff[i] + (j - row) : joff + (row - j);
            if (row < k) g[i] = fma(-(double)Pk[a], dl, g[i]);
          }
          ol = o + 1;
        }
      }
      double amax = 0.0;
#pragma unroll
      for (int i = 0; i < KPL; ++i) amax = fmax(amax, fabs(alpha[i]));
      amax = warp_max(amax);
      if (prof) { const long long t1 = clock64(); c_sw += t1 - t0; t0 = t1; }
      if (maxd <= tol * fmax(1.0, amax)) { ++sweep; break; }
      bool stable = true;
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        const unsigned cm = __ballot_sync(0xffffffffu, alpha[slot] != 0.0);
        stable &= cm == smask[slot];
        smask[slot] = cm;
      }
      ++since_jump;
      if (sweep + 1 < kAsWarm || (!stable && since_jump < kAsForce)) continue;
      since_jump = 0;
      // ---- jump: exact solve on the current face, with line search ----
      int n = 0;
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        const unsigned msk = __ballot_sync(0xffffffffu, alpha[slot] != 0.0);
        const int pos = n + __popc(msk & ((1u << lane) - 1u));
        if (alpha[slot] != 0.0 && pos < nmax) {
          sidx[pos] = slot * 32 + lane;
          av[pos] = alpha[slot];
        }
        n += __popc(msk);
      }
      if (n == 0 || n > nmax) continue;
      for (int j = lane; j < k; j += 32) anew[j] = 0.0;
      bool moved = false;
      int nls = 0;
      __syncwarp();
      while (n > 0) {
        // A = G_SS + l2 I (packed lower), y = beta_S - l1 sign(a_S)
        for (int e = lane; e < n * (n + 1) / 2; e += 32) {
          int r = (int)((sqrtf(8.f * (float)e + 1.f) - 1.f) * 0.5f);
          while (pl_idx(r, 0) > e) --r;
          while (pl_idx(r + 1, 0) <= e) ++r;
          const int c = e - pl_idx(r, 0);
          Af[e] = (double)packed_get(Pk, sidx[r], sidx[c], k) + (r == c ? l2 : 0.0);
        }
        for (int r = lane; r < n; r += 32) {
          const int j = sidx[r];
          yv[r] = beta[(int64_t)j * m + s] - l1 * (av[r] > 0.0 ? 1.0 : -1.0);
        }
        __syncwarp();
        // Cholesky, left-looking (column c: every row r >= c, rows by lane,
        // takes its dot product with row c over the finished columns q < c:
        // independent shared-memory loads into register accumulators, no
        // read-modify-write chain through shared memory); the diagonal holds
        // 1 / L_cc (the substitutions multiply)
        bool ok = true;
        for (int c = 0; c < n; ++c) {
          const int cb = pl_idx(c, 0);
          double sr[kAsRowsPerLane];
#pragma unroll
          for (int j = 0; j < kAsRowsPerLane; ++j) {
            const int r = c + lane + 32 * j;
            double acc = 0.0;
            if (r < n) {
              const int rb = pl_idx(r, 0);
              acc = Af[rb + c];
#pragma unroll 4
              for (int q = 0; q < c; ++q) acc = fma(-Af[rb + q], Af[cb + q], acc);
            }
            sr[j] = acc;
          }
          const double d = __shfl_sync(0xffffffffu, sr[0], 0);     // row c (lane 0)
          if (!(d > 0.0)) { ok = false; break; }
          const double il = rsqrt(d);
          __syncwarp();
#pragma unroll
          for (int j = 0; j < kAsRowsPerLane; ++j) {
            const int r = c + lane + 32 * j;
            if (r < n) Af[pl_idx(r, c)] = r == c ? il : sr[j] * il;
          }
          __syncwarp();
        }
        if (prof) { ++n_solve; n_sum += n; n_max = max(n_max, n); }
        if (!ok) break;
        // L z = y, then L^T x = z, both column-oriented (rows by lane, no reductions)
        for (int c = 0; c < n; ++c) {
          const double zc = yv[c] * Af[pl_idx(c, c)];
          __syncwarp();
          if (lane == 0) yv[c] = zc;
          for (int r = c + 1 + lane; r < n; r += 32) yv[r] = fma(-Af[pl_idx(r, c)], zc, yv[r]);
          __syncwarp();
        }
        for (int c = n - 1; c >= 0; --c) {
          const int cb = pl_idx(c, 0);
          const double xc = yv[c] * Af[cb + c];
          __syncwarp();
          if (lane == 0) yv[c] = xc;
          for (int r = lane; r < c; r += 32) yv[r] = fma(-Af[cb + r], xc, yv[r]);      // L^T[r][c] = L[c][r]
          __syncwarp();
        }
        // signs agree: the face minimiser is the new point
        bool agree = true;
        double tau = 2.0;
        int rmin = n;
        for (int r = lane; r < n; r += 32) {
          const double a0 = av[r], y = yv[r];
          const bool same = a0 > 0.0 ? y > 0.0 : y < 0.0;
          agree &= same;
          if (!same) {
            const double tr = a0 / (a0 - y);                 // in (0, 1]: where a0 + tr (y - a0) = 0
            if (tr < tau || (tr == tau && r < rmin)) { tau = tr; rmin = r; }
          }
        }
        agree = __all_sync(0xffffffffu, agree);
        moved = true;
        if (agree) {
          for (int r = lane; r < n; r += 32) av[r] = yv[r];
          n_agree += 1;
          break;
        }
        // line search: a_S <- a_S + tau (y - a_S), the first zero crossing
        // (smallest tau, lowest position on ties) leaves the support
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double t2 = __shfl_xor_sync(0xffffffffu, tau, o);
          const int r2 = __shfl_xor_sync(0xffffffffu, rmin, o);
          if (t2 < tau || (t2 == tau && r2 < rmin)) { tau = t2; rmin = r2; }
        }
        __syncwarp();
        for (int r = lane; r < n; r += 32) {
          const double a0 = av[r];
          double na = r == rmin ? 0.0 : fma(tau, yv[r] - a0, a0);
          if (a0 > 0.0 ? !(na > 0.0) : !(na < 0.0)) na = 0.0;   // rounding past zero
          av[r] = na;
        }
        __syncwarp();
        // compact the support (order kept)
        int nn = 0;
        for (int r0 = 0; r0 < n; r0 += 32) {
          const int r = r0 + lane;
          const bool keep = r < n && av[r] != 0.0;
          const double va = keep ? av[r] : 0.0;
          const int ja = keep ? sidx[r] : 0;
          const unsigned msk = __ballot_sync(0xffffffffu, keep);
          __syncwarp();
          if (keep) {
            const int pos = nn + __popc(msk & ((1u << lane) - 1u));
            av[pos] = va;
            sidx[pos] = ja;
          }
          nn += __popc(msk);
          __syncwarp();
        }
        n = nn;
        // line-search budget spent: keep the point reached (the objective
        // only decreased along the way) and let the CD sweeps go on
        if (++nls >= kAsMaxLs) break;
      }
      if (!moved) continue;
      // the jump's point (zeros off the final support) back into the registers
      for (int r = lane; r < n; r += 32) anew[sidx[r]] = av[r];
      __syncwarp();
#pragma unroll
      for (int slot = 0; slot < KPL; ++slot) {
        const int j = slot * 32 + lane;
        if (j < k) alpha[slot] = anew[j];
      }
      __syncwarp();
      // g = beta - G alpha (alpha supported on S)
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const int row = lane + 32 * i;
        double acc = 0.0;
        if (row < k) {
          for (int r = 0; r < n; ++r) acc = fma((double)packed_get(Pk, row, sidx[r], k), av[r], acc);
        }
        g[i] = b[i] - acc;
      }
      __syncwarp();
      if (prof) { const long long t1 = clock64(); c_jump += t1 - t0; t0 = t1; }
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
    if (prof && lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(prof + 84), 1ull);
      atomicAdd(reinterpret_cast<unsigned long long*>(prof + 85), (unsigned long long)sweep);
      atomicAdd(reinterpret_cast<unsigned long long*>(prof + 86), (unsigned long long)n_solve);
      atomicAdd(reinterpret_cast<unsigned long long*>(prof + 87), (unsigned long long)n_sum);
      atomicAdd(reinterpret_cast<unsigned long long*>(prof + 88), (unsigned long long)c_sw);
      atomicAdd(reinterpret_cast<unsigned long long*>(prof + 89), (unsigned long long)c_jump);
      atomicMax(prof + 90, (long long)n_max);
      atomicAdd(reinterpret_cast<unsigned long long*>(prof + 91), (unsigned long long)n_agree);
    }
  }
}

}  // namespace somf
