// bcd_shard.cuh -- (a4) Alg. 4 on a ROW SHARD: the
// same simultaneous-threshold rounds as bcd_newton.cuh, but every grid-wide
// sum also has to cross the ranks, so each round is its own kernel and the
// caller's reducer (an allreduce over the ranks; NCCL in bench.py) runs
// between them:
//
//   k_shard_init     atom order, per-atom parameters, Cbar in pi order    (1 CTA)
//   k_shard_setup    per row: D_M and R = P Bbar - P D Cbar in pi order,
//                    radius sums ||P d_j||                        (rows)
//       reducer(radius sums, SUM)
//   repeat:
//     k_shard_round  per row: the recurrence with the current thresholds
//                    (thread per row, R in shared memory), per-atom sums
//                    (count, S1, S2, min above, max below)               (rows)
//       reducer(sums, SUM); reducer(min, MIN); reducer(max, MAX)
//     k_shard_update the Michelot step of every atom, convergence flag    (1 CTA)
//     host reads the flag every kShBatch rounds (rounds after convergence
//     are no-ops): one host synchronisation per kShBatch rounds
//   k_shard_finish   D_M rows back in atom order; slack norms, warm starts (rows)
//
// Every rank runs the identical update on identical reduced sums, so the
// thresholds (and the replicated n_j) stay identical across ranks.
#pragma once
#include "common.cuh"
#include "bcd_newton.cuh"

namespace somf {

// fp64 grid sums of one rank's rows (the rank's total is then allreduced:
// every rank receives the same reduced value, so replicated decisions agree)
__device__ __forceinline__ void nt_red_add(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

constexpr int kShMaxK = 256;
constexpr int kShBatch = 8;     // rounds between two host reads of the convergence flag
// "no element" for the min-above reduction: +inf bits (so the u32 MIN over
// ranks is also a valid int32 MIN for the collectives, all values >= 0)
constexpr unsigned kShNone = 0x7f800000u;

struct ShState {            // device arrays, pi order unless stated
  int* jmap;                // k
  int* pinv;                // k (atom -> position)
  float* invc;              // k
  float* vlo;               // k
  float* thf;               // k
  float* scf;               // k
  double* lam;              // k
  double* rho;              // k
  int* mode;                // k
  float* Cpi;               // k x k (pi order)
  float* Dold;              // q_cap x k
  float* Dn;                // q_cap x k
  float* Rini;              // q_cap x k
  double* acc;              // 3k sums (count, S1, S2)
  double* last;             // 3k sums of the last round (slack)
  unsigned* mn;             // k (float bits, MIN over ranks)
  unsigned* mx;             // k (float bits, MAX over ranks)
  double* rho_acc;          // 2k
  int* conv;                // 2: [0] converged (sticky within a step), [1] rounds run
};

__global__ void k_shard_init(ShState S, const int32_t* __restrict__ perm, const double* __restrict__ C64,
                             const float* __restrict__ C32, const double* __restrict__ lam_ws,
                             const double* __restrict__ nslack, int k, double a, double b, int pos) {
  __shared__ double dmax_s;
  const int tid = threadIdx.x;
  if (tid == 0) {
    double dm = 1.0;
    for (int j = 0; j < k; ++j) dm = fmax(dm, C64[(int64_t)j * k + j]);
    dmax_s = dm;
  }
  __syncthreads();
  for (int p = tid; p < k; p += blockDim.x) {
    const int j = perm[p];
    S.jmap[p] = j;
    S.pinv[j] = p;
    const double cjj = C64[(int64_t)j * k + j];
    const bool dead = !(cjj > 1e-12 * dmax_s);                      // R10
    S.invc[p] = dead ? 0.f : (float)(1.0 / cjj);
    S.vlo[p] = (pos && !dead) ? 0.f : -INFINITY;
    const double lw = dead ? 0.0 : lam_ws[j];
    S.lam[p] = lw;
    S.mode[p] = dead ? kModeDead : (lw > 0.0 ? kModeShrink : kModeCopy);
    S.thf[p] = lw > 0.0 ? (float)(a * lw) : 0.f;
    S.scf[p] = (float)(1.0 / (1.0 + b * lw));
    S.rho[p] = nslack[j];                                            // n_{t-1}; rho after the radius sums
  }
  __syncthreads();
  for (int e = tid; e < k * k; e += blockDim.x) {
    const int p = e / k, l = e % k;
    S.Cpi[e] = C32[(int64_t)S.jmap[p] * k + S.jmap[l]];
  }
  for (int e = tid; e < 3 * k; e += blockDim.x) S.acc[e] = 0.0;
  for (int e = tid; e < 2 * k; e += blockDim.x) S.rho_acc[e] = 0.0;
  for (int e = tid; e < k; e += blockDim.x) {
    S.mn[e] = kShNone;
    S.mx[e] = 0u;
  }
  if (tid == 0) S.conv[0] = S.conv[1] = 0;
}

// thread per masked row: D_M and R in pi order; radius partial sums
__global__ void k_shard_setup(ShState S, const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev,
                              const float* __restrict__ D, const float* __restrict__ Bbar, int k, int kp) {
  const int64_t q = *q_dev;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m < q) {
    const float* drow = D + (int64_t)idx[m] * kp;
    const float* brow = Bbar + (int64_t)idx[m] * kp;
    float* dold = S.Dold + m * k;
    float* rini = S.Rini + m * k;
    for (int p = 0; p < k; ++p) dold[p] = drow[S.jmap[p]];
    for (int p = 0; p < k; ++p) {
      float acc = brow[S.jmap[p]];
      for (int l = 0; l < k; ++l) acc = fmaf(-dold[l], S.Cpi[(int64_t)l * k + p], acc);
      rini[p] = acc;
    }
  }
  // radius sums: one atom per thread of the block, over the block's rows
  __syncthreads();
  const int64_t r0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t r1 = q < r0 + (int64_t)blockDim.x ? q : r0 + (int64_t)blockDim.x;
  for (int p = threadIdx.x; p < k; p += blockDim.x) {
    double d1 = 0.0, d2 = 0.0;
    for (int64_t r = r0; r < r1; ++r) {
      const double d = S.Dold[r * k + p];
      d1 += fabs(d);
      d2 += d * d;
    }
    if (r1 > r0) {
      nt_red_add(S.rho_acc + 2 * p, d1);
      nt_red_add(S.rho_acc + 2 * p + 1, d2);
    }
  }
}

__global__ void k_shard_rho(ShState S, int k, double a, double b) {
  for (int p = threadIdx.x; p < k; p += blockDim.x)
    S.rho[p] = fmax(0.0, S.rho[p] + a * S.rho_acc[2 * p] + 0.5 * b * S.rho_acc[2 * p + 1]);   // P:860, R9
}

// one round of the recurrence: thread per row, R and v in shared memory
// smem: blockDim x (k + 1) floats (R) + blockDim x (k + 1) floats (v)
__global__ void k_shard_round(ShState S, const int64_t* __restrict__ q_dev, int k, double a) {
  // the host checks convergence only every few rounds: rounds after it are
  // no-ops (their sums stay zero; the update below skips them too)
  if (*(volatile int*)S.conv) return;
  extern __shared__ float sh_smem[];
  const int LD = k + 1;
  float* R = sh_smem;                               // rows x LD
  float* V = sh_smem + (size_t)blockDim.x * LD;     // rows x LD
  const int64_t q = *q_dev;
  const int64_t r0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t rem = q - r0;
  const int nr = rem <= 0 ? 0 : (rem < (int64_t)blockDim.x ? (int)rem : (int)blockDim.x);
  const int t = threadIdx.x;
  if (t < nr) {
    const int64_t m = r0 + t;
    float* Rr = R + (size_t)t * LD;
    float* Vr = V + (size_t)t * LD;
    const float* dold = S.Dold + m * k;
    float* dn = S.Dn + m * k;
    for (int p = 0; p < k; ++p) Rr[p] = S.Rini[m * k + p];
    for (int p = 0; p < k; ++p) {
      const float d0 = dold[p];
      const float u = fmaf(Rr[p], S.invc[p], d0);
      const float v = fmaxf(u, S.vlo[p]);
      const float d = copysignf(fmaxf(fabsf(v) - S.thf[p], 0.f) * S.scf[p], v);
      Vr[p] = v;
      dn[p] = d;
      const float delta = d - d0;
      if (delta != 0.f) {
        const float* crow = S.Cpi + (int64_t)p * k;
        for (int l = p + 1; l < k; ++l) Rr[l] = fmaf(-delta, crow[l], Rr[l]);
      }
    }
  }
  __syncthreads();
  for (int p = t; p < k; p += blockDim.x) {
    // exact test |v| > a lambda in fp32: |v| > round_down(a lambda) (as bcd_newton.cuh)
    const double th = a * S.lam[p];
    const bool thr_zero = !(th > 0.0);
    const float thf = thr_zero ? 0.f : __double2float_rd(th);
    double cnt = 0.0, s1 = 0.0, s2 = 0.0;
    unsigned mn = kShNone, mx = 0u;
    for (int r = 0; r < nr; ++r) {
      const float av = fabsf(V[(size_t)r * LD + p]);
      if (av > thf) {
        cnt += 1.0;
        s1 += av;
        s2 += (double)av * av;
        mn = min(mn, __float_as_uint(av));
      } else {
        mx = max(mx, __float_as_uint(av));
      }
    }
    if (nr > 0) {
      if (cnt > 0.0) {
        nt_red_add(S.acc + 3 * p, cnt);
        nt_red_add(S.acc + 3 * p + 1, s1);
        nt_red_add(S.acc + 3 * p + 2, s2);
        atomicMin(S.mn + p, mn);
      }
      if (mx) atomicMax(S.mx + p, mx);
    }
  }
}

// the Michelot step of every atom (identical on every rank); convergence flag
__global__ void k_shard_update(ShState S, int k, double a, double b, int round, int sticky) {
  if (sticky && *(volatile int*)S.conv) return;        // converged in an earlier round of this step
  int conv = 1;
  for (int p = threadIdx.x; p < k; p += blockDim.x) {
    const double cnt = S.acc[3 * p], S1 = S.acc[3 * p + 1], S2 = S.acc[3 * p + 2];
    const double mnv = cnt > 0.0 ? (double)__uint_as_float(S.mn[p]) : INFINITY;
    const double mxv = (double)__uint_as_float(S.mx[p]);
    int nmode;
    double nlam;
    const int cp = nt_atom_update(a, b, S.rho[p], cnt, S1, S2, mnv, mxv, S.mode[p], S.lam[p], &nmode, &nlam,
                                  kNtLamTol, round >= kNtRelaxRound);
    conv &= cp;
    if (cp) {                 // converged atoms keep their parameters (as k_bcd_newton)
      nlam = S.lam[p];
      nmode = S.mode[p];
    }
    S.last[3 * p] = cnt;
    S.last[3 * p + 1] = S1;
    S.last[3 * p + 2] = S2;
    S.lam[p] = nlam;
    S.mode[p] = nmode;
    S.thf[p] = nmode == kModeShrink ? (float)(a * nlam) : 0.f;
    S.scf[p] = nmode == kModeShrink ? (float)(1.0 / (1.0 + b * nlam)) : nmode == kModeZero ? 0.f : 1.f;
    S.acc[3 * p] = S.acc[3 * p + 1] = S.acc[3 * p + 2] = 0.0;
    S.mn[p] = kShNone;
    S.mx[p] = 0u;
  }
  conv = __syncthreads_and(conv);
  if (threadIdx.x == 0) {
    S.conv[0] = conv;
    S.conv[1] += 1;
  }
}

// D_M rows back (the last round's d, atom order); n_j and warm starts
__global__ void k_shard_finish(ShState S, const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev,
                               float* __restrict__ D, int k, int kp, double a, double b,
                               double* __restrict__ nslack, double* __restrict__ lam_ws) {
  const int64_t q = *q_dev;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m < q) {
    float* drow = D + (int64_t)idx[m] * kp;
    for (int j = 0; j < k; ++j) drow[j] = S.Dn[m * k + S.pinv[j]];
  }
  if (blockIdx.x == 0) {
    for (int p = threadIdx.x; p < k; p += blockDim.x) {
      const int mode = S.mode[p];
      if (mode == kModeDead) continue;
      const int j = S.jmap[p];
      // the mode / lambda the last round ran with were replaced by the update:
      // at convergence both agree to kNtLamTol
      nslack[j] = S.rho[p] - nt_norm_d(a, b, mode, S.lam[p], S.last[3 * p], S.last[3 * p + 1], S.last[3 * p + 2]);
      lam_ws[j] = S.lam[p];
    }
  }
}

// ---------------------------------------------------------------------------
// Sharded projection of D_0 onto C (somf_set_components, R15): the same
// Michelot rounds over the ranks with radius 1 for every atom (atom order).
// ---------------------------------------------------------------------------
__global__ void k_proj_init(ShState S, int k) {
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    S.rho[j] = 1.0;
    S.lam[j] = 0.0;
    S.mode[j] = kModeCopy;
    S.acc[3 * j] = S.acc[3 * j + 1] = S.acc[3 * j + 2] = 0.0;
    S.mn[j] = kShNone;
    S.mx[j] = 0u;
  }
}

// one CTA per atom: sums of the |v| above a lambda_j over my rows
__global__ void k_proj_stats(ShState S, const float* __restrict__ D, int64_t rows, int kp, double a, int pos) {
  __shared__ double red_s[3 * 32];
  __shared__ unsigned mm_s[2 * 32];
  const int j = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double th = a * S.lam[j];
  const float thf = th > 0.0 ? __double2float_rd(th) : 0.f;
  double cnt = 0.0, s1 = 0.0, s2 = 0.0;
  unsigned mn = kShNone, mx = 0u;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    float v = D[i * kp + j];
    if (pos) v = fmaxf(v, 0.f);
    const float av = fabsf(v);
    if (av > thf) {
      cnt += 1.0;
      s1 += av;
      s2 += (double)av * av;
      mn = min(mn, __float_as_uint(av));
    } else {
      mx = max(mx, __float_as_uint(av));
    }
  }
  cnt = warp_sum(cnt);
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    red_s[3 * w] = cnt;
    red_s[3 * w + 1] = s1;
    red_s[3 * w + 2] = s2;
    mm_s[2 * w] = mn;
    mm_s[2 * w + 1] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < nw; ++i) {
      cnt += red_s[3 * i];
      s1 += red_s[3 * i + 1];
      s2 += red_s[3 * i + 2];
      mn = min(mn, mm_s[2 * i]);
      mx = max(mx, mm_s[2 * i + 1]);
    }
    S.acc[3 * j] = cnt;
    S.acc[3 * j + 1] = s1;
    S.acc[3 * j + 2] = s2;
    S.mn[j] = mn;
    S.mx[j] = mx;
  }
}

// d = Proj(v) with the converged thresholds; n_j = 1 - ||d_j||
__global__ void k_proj_apply(ShState S, float* __restrict__ D, int64_t rows, int kp, int k, double a, double b,
                             int pos, double* __restrict__ nslack) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < rows * k) {
    const int64_t i = e / k;
    const int j = (int)(e % k);
    float v = D[i * kp + j];
    if (pos) v = fmaxf(v, 0.f);
    const int mode = S.mode[j];
    const double lam = S.lam[j];
    float d = v;
    if (mode == kModeZero) d = 0.f;
    else if (mode == kModeShrink) d = copysignf((float)(fmax(fabs((double)v) - a * lam, 0.0) / (1.0 + b * lam)), v);
    D[i * kp + j] = d;
  }
  if (blockIdx.x == 0)
    for (int j = threadIdx.x; j < k; j += blockDim.x)
      nslack[j] = 1.0 - nt_norm_d(a, b, S.mode[j], S.lam[j], S.last[3 * j], S.last[3 * j + 1], S.last[3 * j + 2]);
}

}  // namespace somf
