// bbar.cuh -- (a3) surrogate statistic on the masked rows, Eq. (somf_partial)
// P:602 (batch mean R4), v2:
//   Bbar[g_m][a] <- (1 - w) Bbar[g_m][a] + (w / eta) sum_s X[m][s] A[a][s]
// for the q masked rows m (g_m = idx[m]) -- or all rows (mode FULL).
//
// Persistent: grid = #SMs, CTA b owns rows [q b / G, q (b+1) / G) and walks
// them in passes of 8 RT rows.  Warp w owns RT rows of the pass; lane l owns
// atoms l, l+32, ... (KC per lane), so the X values are warp broadcasts (read
// 4 columns at a time) and the A^T values and the Bbar row updates are
// coalesced along the atoms.  eta is streamed in chunks of 32 columns: the
// gathered X rows (16-byte cp.async; requires eta % 4 == 0, ldx % 4 == 0 and
// a 16-byte aligned X, checked by the host) and the A^T chunk are double
// buffered.
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kBbThreads = 256;
constexpr int kBbWarps = kBbThreads / 32;
constexpr int kBbSC = 32;                 // eta columns per chunk

__device__ __forceinline__ void bb_cp_async16(void* smem_dst, const void* gmem_src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(gmem_src), "r"(n) : "memory");
}
__device__ __forceinline__ void bb_cp_async4(void* smem_dst, const void* gmem_src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int n = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(gmem_src), "r"(n) : "memory");
}

template <int KC, int RT, bool kGather, bool kXCompact>
__global__ void __launch_bounds__(kBbThreads)
k_bbar_v2(const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev, const float* __restrict__ X,
          int64_t ldx, int eta, const float* __restrict__ A, int k, float* __restrict__ Bbar, int kp,
          const double* __restrict__ w_dev) {
  constexpr int TR = kBbWarps * RT, KA = 32 * KC, SC = kBbSC;
  extern __shared__ __align__(16) float bb_smem[];
  float* Xs = bb_smem;                          // [2][TR][SC]
  float* As = bb_smem + 2 * TR * SC;            // [2][SC][KA]
  __shared__ int grow[TR];
  const int64_t q = *q_dev;
  const double keepd = w_dev[kCoefKeep], gb = w_dev[kCoefGainB];
  const float keep = (float)keepd, add = (float)(gb / eta);
  const int G = gridDim.x;
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nsc = (eta + SC - 1) / SC;

  for (int64_t r0 = lo; r0 < hi; r0 += TR) {
    const int nrow = (int)(hi - r0 < (int64_t)TR ? hi - r0 : (int64_t)TR);
    __syncthreads();
    for (int r = tid; r < TR; r += kBbThreads) grow[r] = r < nrow ? (kGather ? idx[r0 + r] : (int)(r0 + r)) : 0;
    __syncthreads();
    auto load = [&](int sc, int buf) {
      const int s0 = sc * SC;
      float* xb = Xs + buf * TR * SC;
      for (int e = tid; e < TR * (SC / 4); e += kBbThreads) {
        const int r = e / (SC / 4), c = e % (SC / 4);
        const bool ok = r < nrow && s0 + 4 * c < eta;
        const int64_t xr = kXCompact ? r0 + r : (int64_t)grow[r];
        bb_cp_async16(xb + r * SC + 4 * c, ok ? X + xr * ldx + s0 + 4 * c : X, ok);
      }
      float* ab = As + buf * SC * KA;
      for (int e = tid; e < SC * KA; e += kBbThreads) {
        const int a = e / SC, s = e % SC;      // coalesced along s in A (k x eta row-major)
        const bool ok = a < k && s0 + s < eta;
        bb_cp_async4(ab + s * KA + a, ok ? A + (int64_t)a * eta + s0 + s : A, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    float acc[RT][KC];
#pragma unroll
    for (int j = 0; j < RT; ++j)
#pragma unroll
      for (int c = 0; c < KC; ++c) acc[j][c] = 0.f;
    load(0, 0);
    for (int sc = 0; sc < nsc; ++sc) {
      const int buf = sc & 1;
      if (sc + 1 < nsc) {
        load(sc + 1, buf ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncthreads();
      const float* xb = Xs + buf * TR * SC + wid * RT * SC;
      const float* ab = As + buf * SC * KA + lane;
#pragma unroll 2
      for (int s4 = 0; s4 < SC / 4; ++s4) {
        float av[4][KC];
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int c = 0; c < KC; ++c) av[t][c] = ab[(4 * s4 + t) * KA + 32 * c];
#pragma unroll
        for (int j = 0; j < RT; ++j) {
          const float4 x = *reinterpret_cast<const float4*>(xb + j * SC + 4 * s4);
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            acc[j][c] = fmaf(x.x, av[0][c], acc[j][c]);
            acc[j][c] = fmaf(x.y, av[1][c], acc[j][c]);
            acc[j][c] = fmaf(x.z, av[2][c], acc[j][c]);
            acc[j][c] = fmaf(x.w, av[3][c], acc[j][c]);
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int j = 0; j < RT; ++j) {
      const int r = wid * RT + j;
      if (r >= nrow) continue;
      float* brow = Bbar + (int64_t)grow[r] * kp;
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const int a = lane + 32 * c;
        if (a < k) brow[a] = fmaf(keep, brow[a], add * acc[j][c]);
      }
    }
  }
}

}  // namespace somf

namespace somf {

// ---------------------------------------------------------------------------
// v3: one CTA per SM stages its WHOLE slice of masked X rows and the
// transposed codes A^T (eta x kp, written by the code solver) with 16-byte
// cp.async in two commit groups (A^T + first half of the rows, then the second
// half), so every gather is in flight at once (the gather is latency-bound
// otherwise); warp w owns rows w, w+8, ..., lane l atoms l, l+32, ...
// ---------------------------------------------------------------------------
// Optional fold of the Cbar update (Eq. somf_partial; k_cbar_finalize):
// Cbar <- (1 - w) Cbar + (w / eta) sum_b cpart_b, each CTA a slice of the k x k
// entries, partials added in block order (deterministic), so the step needs
// no separate launch for it.
struct CbarFold {
  const double* cpart;      // nparts x k x k (null: no fold)
  int nparts, kk;
  double* C64;
  float* C32;
  const double* A64;        // k x eta codes: fold sum_s a_s a_s^T from them directly (cpart unused)
  int k, eta;
};

template <int KC, int RT, bool kXCompact>
__global__ void __launch_bounds__(kBbThreads, 1)
k_bbar_v3(const int32_t* __restrict__ idx, const int64_t* __restrict__ q_dev, const float* __restrict__ X,
          int64_t ldx, int eta, const float* __restrict__ AT, int kp, int k, float* __restrict__ Bbar,
          const double* __restrict__ w_dev, int seg_rows, CbarFold cf) {
  static_assert(RT % 2 == 0, "RT even: the two halves of the segment are compile-time row ranges");
  constexpr int KA = 32 * KC, SEG = kBbWarps * RT, HALF = SEG / 2;
  extern __shared__ __align__(16) float b3_smem[];
  float* ATs = b3_smem;                               // eta x KA
  float* Xs = ATs + (size_t)eta * KA;                 // SEG x eta (rows >= n zero)
  __shared__ int grow[SEG];
  const int64_t q = *q_dev;
  const double keepd = w_dev[kCoefKeep], gb = w_dev[kCoefGainB], gc = w_dev[kCoefGainC];
  const float keep = (float)keepd, add = (float)(gb / eta);
  const int G = gridDim.x;
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int ce = eta / 4, ck = kp / 4;
  for (int e = tid; e < eta * ck; e += kBbThreads) {
    const int s = e / ck, c = e % ck;
    bb_cp_async16(ATs + (size_t)s * KA + 4 * c, AT + (int64_t)s * kp + 4 * c, true);
  }
  if (cf.cpart) {
    // my slice of the Cbar entries (its loads overlap the A^T staging)
    const int e0 = (int)((int64_t)cf.kk * blockIdx.x / G), e1 = (int)((int64_t)cf.kk * (blockIdx.x + 1) / G);
    for (int e = e0 + tid; e < e1; e += kBbThreads) {
      double s = 0.0;
      for (int bq = 0; bq < cf.nparts; ++bq) s += cf.cpart[(size_t)bq * cf.kk + e];
      const double c = keepd * cf.C64[e] + (gc / eta) * s;
      cf.C64[e] = c;
      cf.C32[e] = (float)c;
    }
  }
  for (int e = tid; e < eta * (KA - kp); e += kBbThreads) {
    const int s = e / (KA - kp), a = kp + e % (KA - kp);
    ATs[(size_t)s * KA + a] = 0.f;
  }
  for (int64_t sb = lo; sb < hi; sb += SEG) {
    const int n = (int)(hi - sb < (int64_t)SEG ? hi - sb : (int64_t)SEG);
    __syncthreads();
    for (int r = tid; r < SEG; r += kBbThreads) grow[r] = r < n ? idx[sb + r] : 0;
    __syncthreads();
    // rows [0, HALF) then [HALF, SEG): two commit groups, every load in flight
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      for (int e = tid; e < HALF * ce; e += kBbThreads) {
        const int r = part * HALF + e / ce, c = e % ce;
        const bool ok = r < n;
        const int64_t xr = kXCompact ? sb + r : (int64_t)grow[r];
        bb_cp_async16(Xs + (size_t)r * eta + 4 * c, ok ? X + xr * ldx + 4 * c : X, ok);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // the old Bbar values of my rows, loaded up front (their latency overlaps the FMAs)
    float bold[RT][KC];
#pragma unroll
    for (int j = 0; j < RT; ++j) {
      const int r = wid + 8 * j;
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const int a = lane + 32 * c;
        bold[j][c] = (r < n && a < k) ? Bbar[(int64_t)grow[r] * kp + a] : 0.f;
      }
    }
    float acc[RT][KC];
#pragma unroll
    for (int j = 0; j < RT; ++j)
#pragma unroll
      for (int c = 0; c < KC; ++c) acc[j][c] = 0.f;
#pragma unroll
    for (int part = 0; part < 2; ++part) {
      if (part == 0) asm volatile("cp.async.wait_group 1;" ::: "memory");
      else asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      const float* ab = ATs + lane;
      for (int s4 = 0; s4 < ce; ++s4) {
        float av[4][KC];
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int c = 0; c < KC; ++c) av[t][c] = ab[(size_t)(4 * s4 + t) * KA + 32 * c];
#pragma unroll
        for (int jj = 0; jj < RT / 2; ++jj) {
          const int j = part * (RT / 2) + jj;
          const int r = wid + 8 * j;      // j in [p RT/2, (p+1) RT/2)  <=>  r in [p HALF, (p+1) HALF)
          const float4 x = *reinterpret_cast<const float4*>(Xs + (size_t)r * eta + 4 * s4);
#pragma unroll
          for (int c = 0; c < KC; ++c) {
            acc[j][c] = fmaf(x.x, av[0][c], acc[j][c]);
            acc[j][c] = fmaf(x.y, av[1][c], acc[j][c]);
            acc[j][c] = fmaf(x.z, av[2][c], acc[j][c]);
            acc[j][c] = fmaf(x.w, av[3][c], acc[j][c]);
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < RT; ++j) {
      const int r = wid + 8 * j;
      if (r >= n) continue;
      float* brow = Bbar + (int64_t)grow[r] * kp;
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const int a = lane + 32 * c;
        if (a < k) brow[a] = fmaf(keep, bold[j][c], add * acc[j][c]);
      }
    }
  }
}

}  // namespace somf
