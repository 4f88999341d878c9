// bcd_newton.cuh -- (a4) Alg. 4 with all k projection thresholds
// solved SIMULTANEOUSLY (v5), for k <= 128 and masked rows that fit on chip.
//
// Alg. 4 visits the atoms in the order pi; atom j's update
//   u = d_j + (bbar_j - D c_j) / c_jj ,  d_j <- Proj(u; rho_j)
// depends on the atoms before it through D, and its projection needs ONE
// scalar of the whole column: the threshold theta_j = a lambda_j of
//   d_i = sign(v_i) max(|v_i| - a lambda_j, 0) / (1 + b lambda_j)     (R17).
// Given ALL thresholds, every masked row runs the whole recurrence on its own
// (no communication).  So instead of one grid reduction per atom (v1/v2), this
// kernel iterates rounds:
//   1. every row runs the full recurrence with the current lambda_1..k (groups
//      of T lanes own M rows, the prescaled residual in registers, the atom
//      loop fully unrolled in permutation order so the arrays stay in
//      registers; see NtRec5);
//   2. ONE grid reduction returns, per atom, the sums (count, S1, S2) of the
//      |v| above its threshold, the smallest |v| above and the largest below;
//   3. every CTA applies the same Michelot step lambda_j <- root of the
//      active-set quadratic (R17) for the set {|v_j| > a lambda_j}.
// The recurrence is triangular (atom j depends only on earlier atoms), so the
// iteration is finite.  It stops when every atom is EXACT (largest |v| below
// <= a lambda' < smallest |v| above: the active set of the new root is the one
// it was computed from) and lambda' equals lambda to kNtLamTol: then the
// round's D is Alg. 4's result to fp32 rounding.  Radii ride on round
// 0's reduction.  Warm start: lambda of the previous iteration.  Identical
// reduced values in every CTA => identical decisions.  The kernel also draws
// the mask of the next iteration (NtArgs draw-ahead fields).
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kNtRing = 3;
constexpr int kProfSlots = 96;      // BCD / ridge profile slots (somf_bcd_phase_cycles)
constexpr int kNtMaxK = 128;        // largest k of the simultaneous-threshold kernel
constexpr int kNtRec = 16;          // 64-bit words per accumulator record (128 bytes)
constexpr int kNtMaxCopies = 16;    // copies of each record (CTA b adds into copy b % ncopy)

// Convergence: every atom exact (its active set reproduces itself) and its
// lambda stable to this relative tolerance between two rounds.  The
// recurrence runs in fp32 (v, d carry ~1e-7 relative rounding); a lambda
// moving by < 1e-5 relative moves d by < 1e-5 of the threshold, inside the 1e-4
// parity tolerance (and the slack norms stay within 1e-5), while a tighter test
// only waits for perturbations of earlier atoms to die out down the chain
// (cfgC r=12: 1e-8 12.1 rounds per step, 1e-6 9.6, 1e-5 8.9; 1e-4 fails the
// slack bound).  SOMF_NT_TOL overrides it.
constexpr double kNtLamTol = 1e-5;

// After this many rounds the exactness test is dropped and an atom converges
// on lambda stability alone.  In exact arithmetic the iteration is finite;
// in floating point an entry |v_i| within rounding of a * lambda_j can make
// the active set flip between two sets whose roots differ by rounding only
// (adding an entry at the threshold moves the root by (|v_i| - theta) / (s + 1)
// ~ 0), which would cycle forever.  The result then differs from the exact
// projection only in entries within rounding of the threshold (the north
// star's support criterion exempts those).  Typical steps converge in <= 16.
constexpr int kNtRelaxRound = 24;

struct NtArgs {
  const int32_t* idx;       // masked local rows (ascending)
  const int64_t* q_dev;
  float* D;                 // rows x kp
  const float* Bbar;        // rows x kp
  const double* C64;        // k x k
  const float* C32;         // k x k
  double* nslack;           // k (atom index)
  double* lam_ws;           // k (atom index): lambda of the previous pass
  const int32_t* perm;      // k (device; used when perm_v is not filled)
  int32_t perm_v[kNtMaxK];  // pi_t by value (drawn on the host, R13), perm_by_value = 1
  int perm_by_value;
  int k, kp;
  double a, b;              // 1 - mu, mu
  int pos;                  // D >= 0
  int cap_rows;             // rows per CTA the shared memory holds (T x cap_rows <= blockDim)
  int ct_in_w;               // Cbar per thread parity fits the staging buffer W
  int part_in_cpi;           // the stats partials (5 H KPT words) fit the Cbar staging area
  int rd_h;                  // threads per atom of the cooperative record read (its 48 rd_h k bytes
                             // reuse the stats partials' area, free after the barrier)
  int max_rounds;
  double lam_tol;           // convergence tolerance on lambda (kNtLamTol)
  // per-atom grid accumulators, 128-byte records (u64 words) so the atomics
  // of different atoms land in different L2 slices, ncopy copies per atom so
  // the same-address chains are ncopy times shorter:
  //   rec[((slot * ncopy + c) * k + p) * kNtRec + w]: w = 0 count, {1,2} S1
  //   limbs, {3,4} S2 limbs (fx_red), 5 = two u32: min |v| above / max |v|
  //   below (float bits); zero (min: all ones) between uses.
  // slots 0..kNtRing-1: the round ring; slot kNtRing: radius sums in S1 / S2
  unsigned long long* rec;
  int ncopy;
  // draw-ahead of iteration t+1 while the CTAs wait on the rounds (null idx_next
  // = off): M_{t+1} (Eq. mt) into idx_next / q_next (per-CTA counts through
  // cnt_next, published before round 0's barrier), t+1 and the coefficients of
  // w_{t+1} = (t+1)^-u into t_next / w_next.  (pi_{t+1} is drawn on the host: perm_v.)
  int32_t* idx_next;
  int64_t* q_next;
  int* cnt_next;            // gridDim.x
  int64_t* t_next;
  double* w_next;
  uint64_t seed, Tthr;
  int64_t tn, row_lo, row_hi;
  StepCoef cf_next;         // coefficients of iteration t+1 (w_{t+1} = (t+1)^-u; common.cuh)
  int cyclic;
  int mbits_off;            // byte offset of the mask-bit scratch in dynamic smem
  unsigned* bar;            // [0] arrivals [1] exits [2] watchdog
  int64_t* nred_out;
  int* err;                 // 2 capacity, 4 round cap
  long long* prof;          // optional: SM cycles per phase, CTA 0 (8 slots), accumulated
  int pdl;                  // launched as a programmatic dependent of the B-bar kernel: the
                            // prologue stages what that kernel does not write (index list, D
                            // rows, warm starts, M_{t+1}) before griddepcontrol.wait
};

// phase clock of CTA 0 (diagnostics only; prof == nullptr disables it)
// (accumulated in shared memory: a global read-modify-write per mark would put
// an L2 round trip on CTA 0's path and distort what it measures; flushed once
// at the end of the kernel)
#define NT_MARK(slot)                                                              \
  do {                                                                             \
    if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) {                           \
      const long long now_ = clock64();                                            \
      prof_s[slot] += now_ - t_mark;                                               \
      t_mark = now_;                                                               \
    }                                                                              \
  } while (0)

enum : int { kModeCopy = 0, kModeZero = 1, kModeShrink = 2, kModeDead = 3 };

__device__ __forceinline__ void nt_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
    if (ld_acquire_gpu(bar) < target) {
      const uint64_t t0 = globaltimer_ns();
      unsigned spins = 0;
      while (ld_acquire_gpu(bar) < target) {
        if ((++spins & 1023u) == 0) {
          if (ld_acquire_gpu(bar + 2)) break;
          if (globaltimer_ns() - t0 > 2000000000ull) { atomicExch(bar + 2, 1u); break; }
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// One Michelot step of atom p from the grid sums over {|v| > a lam} (R17):
// returns 1 when the atom is converged (exact active set, lambda stable).
// Shared by the single-GPU kernel and the row-sharded round kernels.
__device__ __forceinline__ int nt_atom_update(double a, double b, double rho, double cnt, double S1, double S2,
                                              double mnv, double mxv, int mode, double lam, int* nmode_out,
                                              double* nlam_out, double tol = kNtLamTol, bool relax = false) {
  const double th = a * lam;
  int nmode = mode, conv = 1;
  double nlam = lam;
  if (mode == kModeDead) {
    conv = 1;
  } else if (!(rho > 0.0)) {
    nmode = kModeZero;                                               // R11
    conv = mode == kModeZero;
  } else if (!(th > 0.0)) {
    // sums over every nonzero |v|: feasibility, else the root for all of them
    const double Nv = a * S1 + 0.5 * b * S2;
    if (Nv <= rho) {
      nlam = 0.0;
      nmode = kModeCopy;
    } else {
      nlam = enet_lambda(a, b, rho, cnt, S1, S2);
      nmode = nlam > 0.0 ? kModeShrink : kModeCopy;
    }
    // exact when the active set at the new threshold is still "every nonzero"
    const bool exact = nlam == 0.0 || !(a > 0.0) || a * nlam < mnv || relax;
    conv = exact && nmode == mode && fabs(nlam - lam) <= tol * fmax(nlam, 1e-300);
  } else if (!(cnt > 0.0) && a > 0.0 && mxv > 0.0 &&
             a * enet_lambda(a, b, rho, 1.0, mxv, mxv * mxv) >= mxv * (1.0 - 1e-6)) {
    // every |v| is at or below the threshold (d = 0) and even the largest
    // entry alone would sit at the threshold to within rounding: rho is below
    // the resolution of the norm (R11 limit, ~3e-18 seen at cfgE), so d = 0 is
    // the projection to rounding.  (Restarting from the full set here -- the
    // overshoot rule below -- would climb back to the same threshold and cycle.)
    nlam = lam;
    nmode = mode;
    conv = 1;
  } else {
    nlam = enet_lambda(a, b, rho, cnt, S1, S2);
    nmode = nlam > 0.0 ? kModeShrink : kModeCopy;
    const double nth = a * nlam;
    const bool exact = nlam > 0.0 && ((mxv <= nth && nth < mnv) || relax);
    conv = exact && fabs(nlam - lam) <= tol * nlam;
  }
  *nmode_out = nmode;
  *nlam_out = nlam;
  return conv;
}

// ||d_j|| after the projection, from the sums of its final round
__device__ __forceinline__ double nt_norm_d(double a, double b, int mode, double lam, double cnt, double S1,
                                           double S2) {
  const double t = a * lam, opb = 1.0 + b * lam;
  if (mode == kModeCopy) return a * S1 + 0.5 * b * S2;
  if (mode == kModeShrink)
    return a * (S1 - cnt * t) / opb + 0.5 * b * (S2 - 2.0 * t * S1 + cnt * t * t) / (opb * opb);
  return 0.0;
}

__device__ __forceinline__ void nt_rec_reset(unsigned long long* rc) {
#pragma unroll
  for (int w = 0; w < 5; ++w) rc[w] = 0ull;
  rc[5] = 0xffffffffull;          // min above: all ones; max below: 0
}

// the sums of atom p over the ncopy copies of a slot (integers: order-free)
struct NtSums {
  double cnt, S1, S2;
  unsigned mn, mx;
};
__device__ __forceinline__ NtSums nt_read(const unsigned long long* slot0, int ncopy, int k, int p) {
  // two copies per L2 round trip (six 16-byte loads in flight; a full unroll
  // over the copies would cost registers the recurrence needs)
  unsigned long long c = 0, a1 = 0, a2 = 0, b1 = 0, b2 = 0;
  unsigned mn = 0xffffffffu, mx = 0u;
#pragma unroll 1
  for (int c0 = 0; c0 < ncopy; c0 += 2) {
    ulonglong2 v01[2], v23[2], v45[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (c0 + h < ncopy) {
        const unsigned long long* rc = slot0 + ((size_t)(c0 + h) * k + p) * kNtRec;
        v01[h] = __ldcg(reinterpret_cast<const ulonglong2*>(rc));
        v23[h] = __ldcg(reinterpret_cast<const ulonglong2*>(rc + 2));
        v45[h] = __ldcg(reinterpret_cast<const ulonglong2*>(rc + 4));
      } else {
        v01[h] = v23[h] = make_ulonglong2(0ull, 0ull);
        v45[h] = make_ulonglong2(0ull, 0xffffffffull);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      c += v01[h].x;
      a1 += v01[h].y;
      a2 += v23[h].x;
      b1 += v23[h].y;
      b2 += v45[h].x;
      mn = min(mn, (unsigned)(v45[h].y & 0xffffffffull));
      mx = max(mx, (unsigned)(v45[h].y >> 32));
    }
  }
  NtSums r;
  r.cnt = (double)c;
  r.S1 = fx_value(a1, a2);
  r.S2 = fx_value(b1, b2);
  r.mn = mn;
  r.mx = mx;
  return r;
}

// The same sums read COOPERATIVELY: H2 threads per atom each load a strided
// subset of the copies (all of its loads in flight: one L2 round trip instead
// of ncopy / 2), the raw integer partials go to shared memory (part: [H2][k][6]
// u64) and nt_combine adds them (integers: the order does not matter).
__device__ __forceinline__ void nt_read_coop(const unsigned long long* slot0, int ncopy, int k, int H2,
                                             unsigned long long* part) {
  const int tid = threadIdx.x;
  if (tid < H2 * k) {
    const int p = tid % k, h = tid / k;
    unsigned long long c = 0, a1 = 0, a2 = 0, b1 = 0, b2 = 0;
    unsigned mn = 0xffffffffu, mx = 0u;
#pragma unroll 4
    for (int cc = h; cc < ncopy; cc += H2) {
      const unsigned long long* rc = slot0 + ((size_t)cc * k + p) * kNtRec;
      const ulonglong2 v01 = __ldcg(reinterpret_cast<const ulonglong2*>(rc));
      const ulonglong2 v23 = __ldcg(reinterpret_cast<const ulonglong2*>(rc + 2));
      const ulonglong2 v45 = __ldcg(reinterpret_cast<const ulonglong2*>(rc + 4));
      c += v01.x;
      a1 += v01.y;
      a2 += v23.x;
      b1 += v23.y;
      b2 += v45.x;
      mn = min(mn, (unsigned)(v45.y & 0xffffffffull));
      mx = max(mx, (unsigned)(v45.y >> 32));
    }
    unsigned long long* o = part + ((size_t)h * k + p) * 6;
    o[0] = c;
    o[1] = a1;
    o[2] = a2;
    o[3] = b1;
    o[4] = b2;
    o[5] = ((unsigned long long)mx << 32) | mn;
  }
}
__device__ __forceinline__ NtSums nt_combine(const unsigned long long* part, int H2, int k, int p) {
  unsigned long long c = 0, a1 = 0, a2 = 0, b1 = 0, b2 = 0;
  unsigned mn = 0xffffffffu, mx = 0u;
  for (int h = 0; h < H2; ++h) {
    const unsigned long long* o = part + ((size_t)h * k + p) * 6;
    c += o[0];
    a1 += o[1];
    a2 += o[2];
    b1 += o[3];
    b2 += o[4];
    mn = min(mn, (unsigned)(o[5] & 0xffffffffull));
    mx = max(mx, (unsigned)(o[5] >> 32));
  }
  NtSums r;
  r.cnt = (double)c;
  r.S1 = fx_value(a1, a2);
  r.S2 = fx_value(b1, b2);
  r.mn = mn;
  r.mx = mx;
  return r;
}

// ---------------------------------------------------------------------------
// v5 recurrence: a group of T adjacent lanes owns M masked rows.  Thread t of
// a group owns the positions p = i T + t of all M rows: R[m][i] (the residual,
// PRESCALED by 1/c_pp so u = R + d_old) and Do[m][i] (d before this
// pass, constant over the rounds).  Position PP (compile-time, so the arrays
// stay in registers) is owned by t = PP % T; the owner's d - d_old reaches the
// group's other threads with one width-T shuffle per row, then every thread
// updates its own later positions of its M rows with the prescaled Cbar row
// Ct[t][PP][i] = c_{PP, iT+t} / c_{iT+t, iT+t}; each 16-byte shared load of
// Ct serves M rows (shared-memory wavefronts are the limit of this loop).
// Straight-line code over the positions (no per-position branch), so the
// scheduler can overlap one position's chain with the previous one's updates.
// Per-atom parameters: simple case (mu = 0, no D >= 0) the threshold alone
// (theta = +inf zeroes the atom); generic case {theta, 1/(1+b lam), v_lo}.
// Only v is stored: d is a function of v and the round's parameters.
template <bool kGen>
struct NtPar;
template <>
struct NtPar<false> {
  float th;
  __device__ __forceinline__ float d_of(float u) const { return copysignf(fmaxf(fabsf(u) - th, 0.f), u); }
  __device__ __forceinline__ float v_of(float u) const { return u; }
};
template <>
struct NtPar<true> {
  float th, sc, vlo, pad;
  __device__ __forceinline__ float v_of(float u) const { return fmaxf(u, vlo); }
  __device__ __forceinline__ float d_of(float u) const {
    const float v = fmaxf(u, vlo);
    return copysignf(fmaxf(fabsf(v) - th, 0.f) * sc, v);
  }
};

template <int KPT, int T, int M, bool kGen, int PP>
struct NtRec5 {
  static constexpr int KT = KPT / T;
  static constexpr int KTS = (KT + 3) & ~3;
  static __device__ __forceinline__ void run(float (&R)[M][KPT / T], const float (&Do)[M][KPT / T], int t,
                                             float* __restrict__ v0, int vstride,
                                             const float* __restrict__ Ct_t, const NtPar<kGen>* __restrict__ par) {
    constexpr int own = PP % T, ii = PP / T;
    {
      const NtPar<kGen> pr = par[PP];
      float delta[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const float u = R[m][ii] + Do[m][ii];        // P:861 (valid in the owner)
        const float v = pr.v_of(u);
        const float d = pr.d_of(u);
        if (t == own) v0[m * vstride + PP] = v;
        delta[m] = __shfl_sync(0xffffffffu, d - Do[m][ii], own, T);
      }
      const float* crow = Ct_t + PP * KTS;
#pragma unroll
      for (int j4 = ii / 4; j4 < KTS / 4; ++j4) {
        const float4 c = *reinterpret_cast<const float4*>(crow + 4 * j4);
        const float cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int i = 4 * j4 + e;
          if (i < KT) {
#pragma unroll
            for (int m = 0; m < M; ++m) {
              if (i > ii) {
                R[m][i] = fmaf(-delta[m], cc[e], R[m][i]);
              } else if (i == ii) {
                const float up = fmaf(-delta[m], cc[e], R[m][i]);
                R[m][i] = t > own ? up : R[m][i];
              }
            }
          }
        }
      }
    }
    NtRec5<KPT, T, M, kGen, PP + 1>::run(R, Do, t, v0, vstride, Ct_t, par);
  }
};
template <int KPT, int T, int M, bool kGen>
struct NtRec5<KPT, T, M, kGen, KPT> {
  static __device__ __forceinline__ void run(float (&)[M][KPT / T], const float (&)[M][KPT / T], int, float*, int,
                                             const float*, const NtPar<kGen>*) {}
};

// ---------------------------------------------------------------------------
// v6 recurrence (M = 1 row per group of T = 1 or 2 threads): each thread owns
// the positions p = i T + t of ONE masked row; R and Do are float2 pairs so
// the rank-1 updates are packed FFMA2 (fma.rn.f32x2: two FMAs per issued
// instruction -- the v5 loop was issue-bound), the prescaled Cbar row
// Ct[t][PP][.] arrives as 16-byte broadcast loads (every thread of a parity
// reads the same row).  T = 1: no shuffles and no redundant owner work.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 nt_ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

template <int KPT, int T, bool kGen, int PP>
struct NtRec6 {
  static constexpr int KT = KPT / T;          // even (KPT is a multiple of 16)
  static constexpr int KTS = (KT + 3) & ~3;
  // d0: the row's d before the pass in shared memory (Dold, position-major
  // within the row); reading it per position keeps the registers for R and
  // the Cbar prefetch (a register copy of d_old starved the load scheduling)
  static __device__ __forceinline__ void run(float2 (&R)[KT / 2], const float* __restrict__ d0, int t,
                                             float* __restrict__ v0, const float* __restrict__ Ct_t,
                                             const NtPar<kGen>* __restrict__ par) {
    constexpr int own = PP % T, ii = PP / T;
    const NtPar<kGen> pr = par[PP];
    const float rii = (ii & 1) ? R[ii >> 1].y : R[ii >> 1].x;
    const float dii = d0[ii * T + t];
    const float u = rii + dii;                     // P:861 (valid in the owner)
    const float v = pr.v_of(u);
    const float d = pr.d_of(u);
    float delta = d - dii;
    if constexpr (T == 1) {
      v0[PP] = v;
    } else {
      if (t == own) v0[PP] = v;
      delta = __shfl_sync(0xffffffffu, delta, own, T);
    }
    const float2 nd = make_float2(-delta, -delta);
    const float* crow = Ct_t + PP * KTS;
#pragma unroll
    for (int j4 = (ii >> 2); j4 < KTS / 4; ++j4) {
      const float4 c = *reinterpret_cast<const float4*>(crow + 4 * j4);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jp = 2 * j4 + h;                 // pair index: local positions 2 jp, 2 jp + 1
        if (2 * jp + 1 < KT && 2 * jp + 1 >= ii) {
          const float2 cc = h ? make_float2(c.z, c.w) : make_float2(c.x, c.y);
          const float2 up = nt_ffma2(nd, cc, R[jp]);
          // element e of the pair: > ii updated; == ii only where the
          // thread's position lies after PP (t > own); < ii unchanged
          const int e0 = 2 * jp, e1 = 2 * jp + 1;
          float x = R[jp].x, y = R[jp].y;
          if (e0 > ii) x = up.x;
          else if (e0 == ii) x = t > own ? up.x : x;
          if (e1 > ii) y = up.y;
          else if (e1 == ii) y = t > own ? up.y : y;
          R[jp] = make_float2(x, y);
        }
      }
    }
    NtRec6<KPT, T, kGen, PP + 1>::run(R, d0, t, v0, Ct_t, par);
  }
};
template <int KPT, int T, bool kGen>
struct NtRec6<KPT, T, kGen, KPT> {
  static __device__ __forceinline__ void run(float2 (&)[KPT / T / 2], const float*, int, float*, const float*,
                                             const NtPar<kGen>*) {}
};

template <int T, int M>
struct NtCfg {
  // >= T x ceil(rows per CTA / M); T = 1 keeps 2 x KPT / 2 float2 per thread in
  // registers, so at most 384 threads (65536 / 384 = 170 registers)
  static constexpr int kThreads = 384;
};

template <bool kGen>
__device__ __forceinline__ NtPar<kGen> nt_make_par(int mode, double a, double b, double lam, float vlo);
template <>
__device__ __forceinline__ NtPar<false> nt_make_par<false>(int mode, double a, double, double lam, float) {
  NtPar<false> p;
  p.th = mode == kModeShrink ? (float)(a * lam) : mode == kModeZero ? INFINITY : 0.f;
  return p;
}
template <>
__device__ __forceinline__ NtPar<true> nt_make_par<true>(int mode, double a, double b, double lam, float vlo) {
  NtPar<true> p;
  p.th = mode == kModeShrink ? (float)(a * lam) : 0.f;
  p.sc = mode == kModeShrink ? (float)(1.0 / (1.0 + b * lam)) : mode == kModeZero ? 0.f : 1.f;
  p.vlo = mode == kModeDead ? -INFINITY : vlo;
  p.pad = 0.f;
  return p;
}

// Rounds: every round runs the recurrence over all atoms with the current
// thresholds; the iteration ends when every atom is exact and its lambda is
// stable (then the round's v and parameters give Alg. 4's D).  (A frozen
// prefix -- skipping converged leading atoms -- was measured not to help:
// at cfgC the atoms converge out of order, the leading converged run stays
// near 0 until the last rounds.)
template <int KPT, int T, int M, bool kGen>
__global__ void __launch_bounds__(NtCfg<T, M>::kThreads, 1)
k_bcd_newton(NtArgs P) {
  constexpr int LD = KPT + 1;                 // odd row stride: conflict-free per-row access
  constexpr int KT = KPT / T, KTS = (KT + 3) & ~3;
  // Cbar block of one thread parity: padded so the T blocks start in
  // different bank groups (one 16-byte load of a quarter warp touches T blocks)
  constexpr int CTS = ((KPT * KTS + 31) & ~31) + 8;
  static_assert(KPT % T == 0, "KPT must be a multiple of T");
  static_assert((M == 2) || (M == 1 && (T == 1 || T == 2)), "v5: M = 2; v6: M = 1 with T = 1 or 2");
  extern __shared__ __align__(16) float nt_smem[];
  __shared__ __align__(16) NtPar<kGen> par_s[2][KPT];
  __shared__ double lam_s[KPT], rho_s[KPT];
  __shared__ float invc_s[KPT], vlo_s[KPT];
  __shared__ int mode_s[KPT], jmap_s[KPT], pinv_s[KPT];
  __shared__ double dmax_s;
  __shared__ double diag_s[KPT], lws_s[KPT], ns_s[KPT];
  __shared__ int mcnt_s;      // selected rows of M_{t+1} in my slice
  __shared__ long long prof_s[kProfSlots];
  const int k = P.k, kp = P.kp;
  if (P.prof && blockIdx.x == 0)
    for (int i = threadIdx.x; i < kProfSlots; i += blockDim.x) prof_s[i] = 0;
  const int nthr = blockDim.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int64_t q = *P.q_dev;
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  int nr = (int)(hi - lo);
  const int cap = P.cap_rows;
  if (nr > cap || T * ((nr + M - 1) / M) > nthr) {
    if (tid == 0) atomicExch(P.err, 2);
    nr = min(cap, (nthr / T) * M);
  }
  // cap rows + 1 spare row (zeros in Dold / Rini, scratch in V) for the threads past nr
  const size_t blk = ((size_t)(cap + 1) * LD + 3) & ~(size_t)3;   // 16-byte aligned sub-arrays
  float* Dold = nt_smem;                        // cap x LD   (pi order)
  float* Rini = Dold + blk;                     // cap x LD   (staged Cbar, then R0 / c_pp)
  float* V = Rini + blk;                        // cap x LD   (v of the last round; staged D rows first)
  float* W = V + blk;                           // cap x LD   (staged Bbar rows; then Ct when it fits)
  float* Cpi = W + blk;                         // k x KPT    Cbar in pi order, zero padded
  float* Ct = P.ct_in_w ? W : Cpi + (size_t)k * KPT;                    // T x CTS
  int* rows_s = reinterpret_cast<int*>(P.ct_in_w ? Cpi + (size_t)k * KPT : Ct + (size_t)T * CTS);
  const double a = P.a, b = P.b;
  if (tid == 0) mcnt_s = 0;
  long long t_mark = clock64();
  // ---- setup: round 1 (independent of the B-bar kernel: with programmatic
  // dependent launch this overlaps its tail) ---------------------------------------
  for (int r = tid; r < nr; r += nthr) rows_s[r] = P.idx[lo + r];
  for (int p = tid; p < k; p += nthr) {
    jmap_s[p] = P.perm_by_value ? P.perm_v[p] : P.perm[p];
    lws_s[p] = P.lam_ws[p];
    ns_s[p] = P.nslack[p];
  }
  __syncthreads();
  // ---- round 2: the masked rows of D (cp.async, every chunk in flight) ----------
  const int c4 = kp / 4;
  for (int e = tid; e < nr * c4; e += nthr) {
    const int row = e / c4, c = e % c4;
    cp_async16(V + (size_t)row * kp + 4 * c, P.D + (int64_t)rows_s[row] * kp + 4 * c);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  // M_{t+1} of my slice of Philox blocks while the rows are in flight
  uint8_t* mbits_s = reinterpret_cast<uint8_t*>(reinterpret_cast<char*>(nt_smem) + P.mbits_off);
  int64_t mb0 = 0;
  int nmb = 0;
  if (P.idx_next) {
    const int64_t b0 = P.row_lo >> 2, nb = ((P.row_hi - 1) >> 2) - b0 + 1;
    mb0 = b0 + nb * blockIdx.x / G;
    nmb = (int)(b0 + nb * (blockIdx.x + 1) / G - mb0);
    int c = 0;
    for (int i = tid; i < nmb; i += nthr) {
      const uint32_t bits = mask_bits(P.seed, (uint64_t)P.tn, mb0 + i, P.row_lo, P.row_hi, P.Tthr);
      mbits_s[i] = (uint8_t)bits;
      c += __popc(bits);
    }
    c = (int)__reduce_add_sync(0xffffffffu, (unsigned)c);
    if (lane == 0 && c) atomicAdd(&mcnt_s, c);
  }
  // ---- round 3: what the B-bar kernel writes (Cbar, the masked Bbar rows) ----------
  if (P.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const bool cstage = (size_t)cap * LD >= (size_t)k * k + 4;
  if (cstage) {
    for (int e = tid; e < (k * k + 3) / 4; e += nthr) cp_async16(Rini + 4 * e, P.C32 + 4 * e);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int e = tid; e < nr * c4; e += nthr) {
    const int row = e / c4, c = e % c4;
    cp_async16(W + (size_t)row * kp + 4 * c, P.Bbar + (int64_t)rows_s[row] * kp + 4 * c);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int p = tid; p < k; p += nthr) diag_s[p] = P.C64[(int64_t)p * k + p];
  __syncthreads();
  if (wid == 0) {
    double dm = 1.0;
    for (int j = lane; j < k; j += 32) dm = fmax(dm, diag_s[j]);
    dm = warp_max(dm);
    if (lane == 0) dmax_s = dm;
  }
  __syncthreads();
  const double dmax = dmax_s;
  for (int p = tid; p < KPT; p += nthr) {
    if (p < k) {
      const int j = jmap_s[p];
      pinv_s[j] = p;
      const double cjj = diag_s[j];
      const bool dead = !(cjj > 1e-12 * dmax);                      // R10
      const double lw = dead ? 0.0 : lws_s[j];
      lam_s[p] = lw;
      rho_s[p] = ns_s[j];         // n_{t-1}^(j); becomes rho_j after round 0
      const int mode = dead ? kModeDead : (lw > 0.0 ? kModeShrink : kModeCopy);
      mode_s[p] = mode;
      invc_s[p] = dead ? 0.f : (float)(1.0 / cjj);
      vlo_s[p] = P.pos ? 0.f : -INFINITY;                            // D >= 0 clamp
      par_s[0][p] = par_s[1][p] = nt_make_par<kGen>(mode, a, b, lw, vlo_s[p]);
    } else {
      mode_s[p] = kModeDead;
      lam_s[p] = 0.0;
      invc_s[p] = 0.f;
      vlo_s[p] = -INFINITY;
      par_s[0][p] = par_s[1][p] = nt_make_par<kGen>(kModeDead, a, b, 0.0, -INFINITY);
    }
  }
  asm volatile("cp.async.wait_group 1;" ::: "memory");     // D rows and Cbar staged
  __syncthreads();
  for (int e = tid; e < k * KPT; e += nthr) {
    const int p = e / KPT, l = e % KPT;
    const int64_t src = (int64_t)jmap_s[p] * k + (l < k ? jmap_s[l] : 0);
    Cpi[e] = l < k ? (cstage ? Rini[src] : __ldg(P.C32 + src)) : 0.f;
  }
  NT_MARK(76);
  asm volatile("cp.async.wait_group 0;" ::: "memory");     // rows staged
  __syncthreads();
  NT_MARK(77);
  for (int e = tid; e < LD; e += nthr) {
    Dold[(size_t)cap * LD + e] = 0.f;
    Rini[(size_t)cap * LD + e] = 0.f;
  }
  for (int e = tid; e < nr * KPT; e += nthr) {
    const int row = e / KPT, p = e % KPT;
    const bool in = p < k;
    const int j = in ? jmap_s[p] : 0;
    Dold[(size_t)row * LD + p] = in ? V[(size_t)row * kp + j] : 0.f;
    Rini[(size_t)row * LD + p] = in ? W[(size_t)row * kp + j] : 0.f;
  }
  __syncthreads();
  // prescaled Cbar per thread parity (W is free now): c_{p,l} / c_{l,l}
  for (int e = tid; e < T * KPT * KTS; e += nthr) {
    const int t = e / (KPT * KTS), rem = e % (KPT * KTS), p = rem / KTS, i = rem % KTS;
    const int l = i * T + t;
    Ct[(size_t)t * CTS + rem] = (i < KT && p < k) ? Cpi[(size_t)p * KPT + l] * invc_s[l] : 0.f;
  }
  NT_MARK(78);
  // R = (P Bbar - P D Cbar) / c_pp: RT rows x 8 positions per item (register tile)
  {
    constexpr int RT = 4;                 // ~2 items per thread at 288 threads
    const int nrb = (nr + RT - 1) / RT, npb = (k + 7) / 8;
    for (int it = tid; it < nrb * npb; it += nthr) {
      const int r0 = (it / npb) * RT, p0 = (it % npb) * 8;
      float acc[RT][8];
#pragma unroll
      for (int i = 0; i < RT; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[i][c] = 0.f;
      for (int l = 0; l < k; ++l) {
        const float4 c0 = *reinterpret_cast<const float4*>(Cpi + (size_t)l * KPT + p0);
        const float4 c1 = *reinterpret_cast<const float4*>(Cpi + (size_t)l * KPT + p0 + 4);
        const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
        for (int i = 0; i < RT; ++i) {
          const float d = Dold[(size_t)min(r0 + i, cap - 1) * LD + l];
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[i][c] = fmaf(d, cv[c], acc[i][c]);
        }
      }
#pragma unroll
      for (int i = 0; i < RT; ++i) {
        const int row = r0 + i;
        if (row >= nr) continue;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int p = p0 + c;
          if (p < k) {
            float* rr = Rini + (size_t)row * LD + p;
            *rr = (*rr - acc[i][c]) * invc_s[p];
          }
        }
      }
    }
  }
  // radii (R9): ||P d_j|| of the column before its update, one warp per atom
  if (nr > 0) {
    const int nwarp = nthr >> 5;
    for (int p = wid; p < k; p += nwarp) {
      double d1 = 0.0, d2 = 0.0;
      for (int row = lane; row < nr; row += 32) {
        const double d = Dold[(size_t)row * LD + p];
        d1 += fabs(d);
        d2 += d * d;
      }
      d1 = warp_sum(d1);
      d2 = warp_sum(d2);
      if (lane == 0) {
        unsigned long long* rr =
            P.rec + (((size_t)kNtRing * P.ncopy + blockIdx.x % P.ncopy) * k + p) * kNtRec;
        const bool ok = fx_red(rr + 1, d1) & fx_red(rr + 3, d2);
        if (!ok) atomicExch(P.err, 6);
      }
    }
  }
  __syncthreads();
  // my rows: M consecutive rows of group g; rows >= nr use the spare row
  const int g = tid / T, tq = tid % T;
  int rowx[M];
#pragma unroll
  for (int m = 0; m < M; ++m) rowx[m] = (g * M + m < nr) ? g * M + m : cap;
  const int vstride = (rowx[M - 1] - rowx[0]);          // 1 row apart unless the tail hits the spare row
  constexpr int KT2 = M == 1 ? KT / 2 : 1;
  float Do[M][KT];
  if constexpr (M != 1) {
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int i = 0; i < KT; ++i) Do[m][i] = Dold[(size_t)rowx[m] * LD + i * T + tq];
  }
  const float* Ct_t = Ct + (size_t)tq * CTS;

  // stats partials (H threads per atom) reuse the Cbar staging area (host checks the size)
  const int H = max(1, nthr / max(k, 1));
  unsigned* pcn = P.part_in_cpi ? reinterpret_cast<unsigned*>(Cpi)
                                : reinterpret_cast<unsigned*>((reinterpret_cast<uintptr_t>(rows_s + cap) + 15) & ~(uintptr_t)15);
  float* ps1 = reinterpret_cast<float*>(pcn + H * KPT);
  float* ps2 = ps1 + H * KPT;
  unsigned* pmn = reinterpret_cast<unsigned*>(ps2 + H * KPT);
  unsigned* pmx = pmn + H * KPT;
  __syncthreads();
  if (P.idx_next && tid == 0) P.cnt_next[blockIdx.x] = mcnt_s;   // before round 0's barrier
  NT_MARK(0);
  unsigned nbar = 0;
  int round = 0, cur = 0;
  constexpr int F = 0;          // (no frozen prefix: every round runs every atom)
  bool done = q == 0;
  if (done && P.idx_next) {
    // empty mask: no rounds, but the draw-ahead below reads every CTA's count
    // of M_{t+1}, published above -- one barrier orders them
    ++nbar;
    nt_barrier(P.bar, nbar * G);
  }
#pragma unroll 1
  while (!done) {
    // ---- 1. the recurrence from the frozen prefix on, T threads x M rows ---------
    {
      // every thread of a warp with rows runs it (the width-T shuffles need
      // converged warps; rows >= nr compute on the spare row's zeros); warps
      // past the rows (launched for the statistics and the setup) skip it
      const bool warp_has_rows = ((tid & ~31) / T) * M < nr;
      if constexpr (M == 1) {
        if (warp_has_rows) {
        float2 R2[KT2];
#pragma unroll
        for (int i = 0; i < KT2; ++i)
          R2[i] = make_float2(Rini[(size_t)rowx[0] * LD + (2 * i) * T + tq],
                              Rini[(size_t)rowx[0] * LD + (2 * i + 1) * T + tq]);
        NtRec6<KPT, T, kGen, 0>::run(R2, Dold + (size_t)rowx[0] * LD, tq, V + (size_t)rowx[0] * LD, Ct_t,
                                     par_s[cur]);
        }
      } else if (warp_has_rows) {
        float R[M][KT];
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int i = 0; i < KT; ++i) R[m][i] = Rini[(size_t)rowx[m] * LD + i * T + tq];
        // rows rowx[0] and rowx[0] + vstride (vstride = LD for consecutive rows; the
        // spare row is its own target when both are past nr)
        NtRec5<KPT, T, M, kGen, 0>::run(R, Do, tq, V + (size_t)rowx[0] * LD,
                                        M > 1 ? vstride * LD : 0, Ct_t, par_s[cur]);
      }
    }
    __syncthreads();
    NT_MARK(1);
    // ---- 2. per-atom statistics over my rows, then one grid reduction -------------
    // H threads per atom sum a strided share of the rows (fp32 over <= cap/H
    // rows, relative error ~1e-6), combined in fixed order.
    const int ring = round % kNtRing;
    const int nact = k - F;
    if (nr > 0) {
      if (tid < H * nact) {
        const int p = F + tid % nact, h = tid / nact;
        const double th = a * lam_s[p];
        // the test is exact: for a float |v| and a double th,
        // |v| > th  <=>  |v| > round_down_to_float(th)
        const float thf = th > 0.0 ? __double2float_rd(th) : 0.f;
        unsigned cnt = 0, mn = 0xffffffffu, mx = 0u;
        float s1 = 0.f, s2 = 0.f;
#pragma unroll 4
        for (int r = h; r < nr; r += H) {
          const float av = fabsf(V[(size_t)r * LD + p]);
          const bool above = av > thf;
          cnt += above;
          s1 += above ? av : 0.f;
          s2 = fmaf(above ? av : 0.f, av, s2);
          mn = above ? min(mn, __float_as_uint(av)) : mn;
          mx = above ? mx : max(mx, __float_as_uint(av));
        }
        pcn[h * KPT + p] = cnt;
        ps1[h * KPT + p] = s1;
        ps2[h * KPT + p] = s2;
        pmn[h * KPT + p] = mn;
        pmx[h * KPT + p] = mx;
      }
      __syncthreads();
      if (tid < nact) {
        const int p = F + tid;
        unsigned cnt = 0, mn = 0xffffffffu, mx = 0u;
        double S1 = 0.0, S2 = 0.0;
        for (int h = 0; h < H; ++h) {
          cnt += pcn[h * KPT + p];
          S1 += (double)ps1[h * KPT + p];
          S2 += (double)ps2[h * KPT + p];
          mn = min(mn, pmn[h * KPT + p]);
          mx = max(mx, pmx[h * KPT + p]);
        }
        unsigned long long* rc = P.rec + (((size_t)ring * P.ncopy + blockIdx.x % P.ncopy) * k + p) * kNtRec;
        unsigned* mm = reinterpret_cast<unsigned*>(rc + 5);
        if (cnt > 0) {
          nt_red_u64(rc, (unsigned long long)cnt);
          const bool ok = fx_red(rc + 1, S1) & fx_red(rc + 3, S2);
          if (!ok) atomicExch(P.err, 6);
          atomicMin(mm, mn);
        }
        if (mx) atomicMax(mm + 1, mx);
      }
    }
    NT_MARK(2);
    ++nbar;
    nt_barrier(P.bar, nbar * G);
    NT_MARK(3);
    {
      // recycle the ring slot of the NEXT-but-one round (every CTA read it in
      // the previous round, before this barrier; it is written again only after
      // the next one): record e by CTA e % G, spread over the grid
      const int rz = (round + 2) % kNtRing;
      for (int e = blockIdx.x + G * tid; e < P.ncopy * k; e += G * nthr)
        nt_rec_reset(P.rec + ((size_t)rz * P.ncopy * k + e) * kNtRec);
    }
    NT_MARK(80);
    // ---- 3. the same Michelot step for every unfrozen atom in every CTA ----------
    int conv = 1, nmode = 0;
    double nlam = 0.0, cnt = 0.0, S1 = 0.0, S2 = 0.0;
    const int p = F + tid;
    const bool act = tid < nact;
    unsigned long long* rdp = reinterpret_cast<unsigned long long*>(pcn);
    if (round == 0) {
      nt_read_coop(P.rec + (size_t)kNtRing * P.ncopy * k * kNtRec, P.ncopy, k, P.rd_h, rdp);
      __syncthreads();
      if (act) {
        const NtSums rs = nt_combine(rdp, P.rd_h, k, p);
        rho_s[p] = fmax(0.0, rho_s[p] + a * rs.S1 + 0.5 * b * rs.S2);     // P:860, R9
      }
      __syncthreads();
    }
    nt_read_coop(P.rec + (size_t)ring * P.ncopy * k * kNtRec, P.ncopy, k, P.rd_h, rdp);
    __syncthreads();
    NT_MARK(81);
    if (act) {
      const NtSums sm = nt_combine(rdp, P.rd_h, k, p);
      cnt = sm.cnt;
      S1 = sm.S1;
      S2 = sm.S2;
      const double mnv = cnt > 0.0 ? (double)__uint_as_float(sm.mn) : INFINITY;
      const double mxv = (double)__uint_as_float(sm.mx);
      conv = nt_atom_update(a, b, rho_s[p], cnt, S1, S2, mnv, mxv, mode_s[p], lam_s[p], &nmode, &nlam, P.lam_tol,
                            round >= kNtRelaxRound);
    }
    // every atom converged: the round's v and parameters are final (a frozen
    // prefix was measured not to help: atoms converge out of order)
    const int Fn = __syncthreads_and(conv) ? k : 0;
    const bool capped = round + 1 >= P.max_rounds && Fn < k;
    if (act) {
      if (p < Fn || capped) {
        // frozen with this round's parameters: slack n_j = rho_j - ||d_j|| from
        // this round's sums, warm start for the next iteration
        if (mode_s[p] != kModeDead && blockIdx.x == 0) {
          const int j = jmap_s[p];
          P.nslack[j] = rho_s[p] - nt_norm_d(a, b, mode_s[p], lam_s[p], cnt, S1, S2);
          P.lam_ws[j] = lam_s[p];
        }
        par_s[cur ^ 1][p] = par_s[cur][p];
      } else if (conv) {
        // converged atoms keep their parameters while others move: the v of
        // the atoms after them then only change when an unconverged atom
        // before them does (no tolerance-level jitter propagating down the
        // chain; at cfgE it kept later atoms from ever settling)
        par_s[cur ^ 1][p] = par_s[cur][p];
      } else {
        lam_s[p] = nlam;
        mode_s[p] = nmode;
        par_s[cur ^ 1][p] = nt_make_par<kGen>(nmode, a, b, nlam, vlo_s[p]);
      }
    }
    // (frozen and padding positions hold the same parameters in both buffers)
    if (P.prof && blockIdx.x == 0) {
      // convergence profile: unconverged atoms per round (slots 8..71)
      const int nun = __syncthreads_count(act && !conv);
      if (tid == 0 && round < 64) prof_s[8 + round] += nun + ((long long)F << 16);   // (F << 16) + unconverged
    }
    NT_MARK(4);
    ++round;
    if (Fn >= k) {
      done = true;
    } else if (capped) {
      if (tid == 0 && blockIdx.x == 0) atomicExch(P.err, 4);
      done = true;
    }
    if (!done) cur ^= 1;
  }
  __syncthreads();
  NT_MARK(5);
  // ---- final D = the v of each atom's final round through its parameters, atom order ----
  // (with the draw-ahead on, the last warp scatters M_{t+1} and stays out of
  // the write-back so the two overlap)
  const int nwarp_all = nthr >> 5;
  const bool ahead = P.idx_next != nullptr && nwarp_all >= 4;
  if (q > 0 && !(ahead && wid == nwarp_all - 1)) {
    const NtPar<kGen>* pr = par_s[cur];
    const int nwarp = ahead ? nwarp_all - 1 : nwarp_all;
    for (int r = wid; r < nr; r += nwarp) {
      float* dst = P.D + (int64_t)rows_s[r] * kp;
      const float* src = V + (size_t)r * LD;
      for (int j = lane; j < k; j += 32) {
        const int pp = pinv_s[j];
        dst[j] = pr[pp].d_of(src[pp]);
      }
    }
  }
  // ---- draw-ahead of t+1: scatter of my slice of M_{t+1}, t+1, w_{t+1} ------------------
  if (P.idx_next) {
    const int nwarp = nthr >> 5;
    if (wid == nwarp - 1) {
      // rows of M_{t+1} before my slice: counts of the CTAs before me (fixed order)
      int64_t off = 0;
      for (int i = lane; i < (int)blockIdx.x; i += 32) off += __ldcg(P.cnt_next + i);
      off = warp_sum(off);
      // lane l scans the blocks [l nmb / 32, (l+1) nmb / 32) of my slice
      const int i0 = nmb * lane / 32, i1 = nmb * (lane + 1) / 32;
      int c = 0;
      for (int i = i0; i < i1; ++i) c += __popc((unsigned)mbits_s[i]);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      int64_t pos = off + incl - c;
      for (int i = i0; i < i1; ++i) {
        const unsigned bits = mbits_s[i];
        for (int l = 0; l < 4; ++l)
          if (bits & (1u << l)) P.idx_next[pos++] = (int32_t)((mb0 + i) * 4 + l - P.row_lo);
      }
      if (blockIdx.x == G - 1 && lane == 31) *P.q_next = pos;
    }
    if (blockIdx.x == 0 && wid == 0 && lane == 0) {
      *P.t_next = P.tn;
      store_coef(P.w_next, P.cf_next);
    }
  }
  // ---- exit: last CTA resets counters and accumulators ------------------------------
  __syncthreads();
  NT_MARK(6);
  if (P.prof && blockIdx.x == 0) {
    __syncthreads();
    if (threadIdx.x == 0) prof_s[7] += 1;
    __syncthreads();
    for (int i = threadIdx.x; i < kProfSlots; i += blockDim.x)
      if (i < 72 || i >= 76) P.prof[i] += prof_s[i];              // (72..75: the ridge solver's)
  }
  if (tid == 0) {
    __threadfence();
    const unsigned old = atomicAdd(P.bar + 1, 1u);
    mcnt_s = old == (unsigned)G - 1;      // (mcnt_s is free now) I am the last CTA out
  }
  __syncthreads();
  if (mcnt_s) {
    __threadfence();
    for (int e = tid; e < (kNtRing + 1) * P.ncopy * k; e += nthr) nt_rec_reset(P.rec + (size_t)e * kNtRec);
    if (tid == 0) {
      if (P.nred_out) *P.nred_out = nbar;
      P.bar[0] = 0u;
      P.bar[1] = 0u;
    }
    __threadfence();
  }
}

}  // namespace somf
