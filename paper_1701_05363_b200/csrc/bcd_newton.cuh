// bcd_newton.cuh -- (a4) Alg. 4 with all k projection thresholds
// solved SIMULTANEOUSLY (v3), for k <= 96 and masked rows that fit on chip.
//
// Alg. 4 visits the atoms in the order pi; atom j's update
//   u = d_j + (bbar_j - D c_j) / c_jj ,  d_j <- Proj(u; rho_j)
// depends on the atoms before it through D, and its projection needs ONE
// scalar of the whole column: the threshold theta_j = a lambda_j of
//   d_i = sign(v_i) max(|v_i| - a lambda_j, 0) / (1 + b lambda_j)     (R17).
// Given ALL thresholds, every masked row runs the whole recurrence on its own
// (no communication).  So instead of one grid reduction per atom (v1/v2), this
// kernel iterates rounds:
//   1. every row runs the full recurrence with the current lambda_1..k
//      (thread per row, residual R = P Bbar - P D Cbar in registers, the atom
//      loop fully unrolled in permutation order so R is indexed statically);
//   2. ONE grid reduction returns, per atom, the sums (count, S1, S2) of the
//      |v| above its threshold, the smallest |v| above and the largest below;
//   3. every CTA applies the same Michelot step lambda_j <- root of the
//      active-set quadratic (R17) for the set {|v_j| > a lambda_j}.
// The recurrence is triangular (atom j depends only on earlier atoms), so once
// atoms 1..j-1 are fixed atom j's set can only shrink (Michelot from a
// superset) and the iteration is finite.  It stops when every atom is EXACT
// (largest |v| below <= a lambda' < smallest |v| above: the active set of the
// new root is the one it was computed from) and lambda' equals lambda to
// kNtLamTol: then the round's D is Alg. 4's result to fp32 rounding.  Radii
// ride on round 0's reduction.  Warm start: lambda of the previous iteration.
// Identical reduced values in every CTA => identical decisions.
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kNtThreads = 384;     // 2 threads per masked row: >= 2 x rows per CTA
constexpr int kNtRing = 3;
// Convergence: every atom exact (its active set reproduces itself) and its
// lambda stable to this relative tolerance between two rounds.  The
// recurrence runs in fp32 (v, d carry ~1e-7 relative rounding), so asking for
// more than ~1e-8 only makes rounding noise of one atom ripple down the
// chain one round per atom.
constexpr double kNtLamTol = 1e-8;

struct NtArgs {
  const int32_t* idx;       // masked local rows (ascending)
  const int64_t* q_dev;
  float* D;                 // rows x kp
  const float* Bbar;        // rows x kp
  const double* C64;        // k x k
  const float* C32;         // k x k
  double* nslack;           // k (atom index)
  double* lam_ws;           // k (atom index): lambda of the previous pass
  const int32_t* perm;      // k
  int k, kp;
  double a, b;              // 1 - mu, mu
  int pos;                  // D >= 0
  int cap_rows;             // rows per CTA the shared memory holds (<= kNtThreads)
  int max_rounds;
  double* acc;              // [kNtRing][k][3]  (zero between uses)
  unsigned* accmm;          // [kNtRing][k][2]  min-above (0xffffffff) / max-below (0)
  double* rho_acc;          // [2k]             (zero between uses)
  unsigned* bar;            // [0] arrivals [1] exits [2] watchdog
  int64_t* nred_out;
  int* err;                 // 2 capacity, 4 round cap
  long long* prof;          // optional: SM cycles per phase, CTA 0 (8 slots), accumulated
};

// phase clock of CTA 0 (diagnostics only; prof == nullptr disables it)
#define NT_MARK(slot)                                                              \
  do {                                                                             \
    if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) {                           \
      const long long now_ = clock64();                                            \
      P.prof[slot] += now_ - t_mark;                                               \
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
                                              double* nlam_out) {
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
    const bool exact = nlam == 0.0 || !(a > 0.0) || a * nlam < mnv;
    conv = exact && nmode == mode && fabs(nlam - lam) <= kNtLamTol * fmax(nlam, 1e-300);
  } else {
    nlam = enet_lambda(a, b, rho, cnt, S1, S2);
    nmode = nlam > 0.0 ? kModeShrink : kModeCopy;
    const double nth = a * nlam;
    const bool exact = nlam > 0.0 && mxv <= nth && nth < mnv;
    conv = exact && fabs(nlam - lam) <= kNtLamTol * nlam;
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

__device__ __forceinline__ void nt_red_add(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// One atom of the recurrence at compile-time position PP (so R[] is indexed
// statically and stays in registers), then the next position.
template <int KPT, int PP>
struct NtRec {
  // __restrict__: the v / d stores of one position must not pin the loads of
  // the next positions (and the Cbar rows) behind them, or no two positions'
  // dependency chains can overlap
  static __device__ __forceinline__ void run(float (&R)[KPT], const float* __restrict__ drow,
                                             float* __restrict__ vrow, float* __restrict__ dnrow,
                                             const float* __restrict__ Cpi, const float* __restrict__ invc_s,
                                             const float* __restrict__ thf_s, const float* __restrict__ scf_s,
                                             const float* __restrict__ vlo_s, int k) {
    if (PP >= k) return;
    // branch-free: copy = (th 0, scale 1), zero = scale 0, dead = (invc 0, copy)
    const float dold = drow[PP];
    const float u = fmaf(R[PP], invc_s[PP], dold);
    const float v = fmaxf(u, vlo_s[PP]);
    const float d = copysignf(fmaxf(fabsf(v) - thf_s[PP], 0.f) * scf_s[PP], v);
    vrow[PP] = v;
    dnrow[PP] = d;
    const float delta = d - dold;
    // rank-1 update of the later positions: straight-line (no delta == 0
    // branch) so ptxas can overlap it with the next position's chain; the
    // Cbar row is read 16 bytes at a time (rows are 16-byte aligned).
    const float4* crow = reinterpret_cast<const float4*>(Cpi + (size_t)PP * KPT);
#pragma unroll
    for (int l4 = (PP + 1) / 4; l4 < KPT / 4; ++l4) {
      const float4 c = crow[l4];
      if (4 * l4 + 0 > PP) R[4 * l4 + 0] = fmaf(-delta, c.x, R[4 * l4 + 0]);
      if (4 * l4 + 1 > PP) R[4 * l4 + 1] = fmaf(-delta, c.y, R[4 * l4 + 1]);
      if (4 * l4 + 2 > PP) R[4 * l4 + 2] = fmaf(-delta, c.z, R[4 * l4 + 2]);
      if (4 * l4 + 3 > PP) R[4 * l4 + 3] = fmaf(-delta, c.w, R[4 * l4 + 3]);
    }
    NtRec<KPT, PP + 1>::run(R, drow, vrow, dnrow, Cpi, invc_s, thf_s, scf_s, vlo_s, k);
  }
};
template <int KPT>
struct NtRec<KPT, KPT> {
  static __device__ __forceinline__ void run(float (&)[KPT], const float*, float*, float*, const float*,
                                             const float*, const float*, const float*, const float*, int) {}
};

// Two threads per row (lanes 2r and 2r+1): the thread of parity t holds the
// residual of the positions p = t (mod 2) in R[p / 2].  Position PP is owned by
// parity PP % 2 (compile-time); the owner's d - d_old reaches its partner with
// one shuffle, then each thread updates its own later positions.  Halves the
// FMAs per thread and doubles the warps that hide the per-position chain.
template <int KPT, int PP>
struct NtRec2 {
  static __device__ __forceinline__ void run(float (&R)[KPT / 2], int par, int pairbase, bool wr,
                                             const float* drow, float* vrow, float* dnrow, const float* Cpi,
                                             const float* invc_s, const float* thf_s, const float* scf_s,
                                             const float* vlo_s, int k) {
    if (PP >= k) return;
    constexpr int own = PP & 1;
    const float dold = drow[PP];
    const float u = fmaf(R[PP / 2], invc_s[PP], dold);                // P:861 (valid in the owner)
    const float v = fmaxf(u, vlo_s[PP]);
    const float d = copysignf(fmaxf(fabsf(v) - thf_s[PP], 0.f) * scf_s[PP], v);
    if (wr && par == own) {
      vrow[PP] = v;
      dnrow[PP] = d;
    }
    const float delta = __shfl_sync(0xffffffffu, d - dold, pairbase | own);
    const float* crow = Cpi + (size_t)PP * KPT;
#pragma unroll
    for (int l2 = PP / 2; l2 < KPT / 2; ++l2) {
      // my position l = 2 l2 + par; update it if it comes after PP
      const float2 c = *reinterpret_cast<const float2*>(crow + 2 * l2);
      const float cl = par ? c.y : c.x;
      const bool later = (2 * l2 + 1 > PP);            // parity-1 position 2 l2 + 1 is later
      const bool later0 = (2 * l2 > PP);               // parity-0 position 2 l2 is later
      if (par ? later : later0) R[l2] = fmaf(-delta, cl, R[l2]);
    }
    NtRec2<KPT, PP + 1>::run(R, par, pairbase, wr, drow, vrow, dnrow, Cpi, invc_s, thf_s, scf_s, vlo_s, k);
  }
};
template <int KPT>
struct NtRec2<KPT, KPT> {
  static __device__ __forceinline__ void run(float (&)[KPT / 2], int, int, bool, const float*, float*, float*,
                                             const float*, const float*, const float*, const float*, const float*,
                                             int) {}
};

template <int KPT>
__global__ void __launch_bounds__(kNtThreads, 1)
k_bcd_newton(NtArgs P) {
  constexpr int LD = KPT + 1;                 // odd row stride: conflict-free per-row access
  extern __shared__ __align__(16) float nt_smem[];
  __shared__ double lam_s[KPT], rho_s[KPT];
  __shared__ float thf_s[KPT], scf_s[KPT], invc_s[KPT], vlo_s[KPT];
  __shared__ int mode_s[KPT], jmap_s[KPT], pinv_s[KPT];
  __shared__ int conv_all_s;
  const int k = P.k, kp = P.kp;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int64_t q = *P.q_dev;
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  int nr = (int)(hi - lo);
  if (nr > P.cap_rows) {
    if (tid == 0) atomicExch(P.err, 2);
    nr = P.cap_rows;
  }
  const int cap = P.cap_rows;
  const size_t blk = ((size_t)cap * LD + 3) & ~(size_t)3;   // 16-byte aligned sub-arrays
  float* Dold = nt_smem;                        // cap x LD   (pi order)
  float* Rini = Dold + blk;                     // cap x LD
  float* V = Rini + blk;                        // cap x LD   (v of the last round)
  float* Dn = V + blk;                          // cap x LD   (d of the last round = the result)
  float* Cpi = Dn + blk;                        // k x KPT    Cbar in pi order, zero padded
  double* part = reinterpret_cast<double*>(Cpi + (size_t)k * KPT);   // stats partials (see below)
  const double a = P.a, b = P.b;

  int* rows_s = reinterpret_cast<int*>(part + 3 * (size_t)max(1, kNtThreads / max(k, 1)) * KPT +
                                       (size_t)max(1, kNtThreads / max(k, 1)) * KPT);   // cap
  __shared__ double dmax_s;
  __shared__ double diag_s[KPT], lws_s[KPT], ns_s[KPT];
  long long t_mark = clock64();
  // ---- setup: round 1 (independent loads) ------------------------------------------
  // Cbar (fp32, atom order) -> Rini as a staging buffer when it fits, the row
  // indices, the atom order and the per-atom scalars, all in flight at once
  const bool cstage = (size_t)cap * LD >= (size_t)k * k + 4;
  if (cstage) {
    for (int e = tid; e < (k * k + 3) / 4; e += kNtThreads) cp_async16(Rini + 4 * e, P.C32 + 4 * e);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  for (int r = tid; r < nr; r += kNtThreads) rows_s[r] = P.idx[lo + r];
  for (int p = tid; p < k; p += kNtThreads) {
    jmap_s[p] = P.perm[p];
    diag_s[p] = P.C64[(int64_t)p * k + p];
    lws_s[p] = P.lam_ws[p];
    ns_s[p] = P.nslack[p];
  }
  __syncthreads();
  // ---- round 2: the masked rows of D and Bbar (cp.async, every chunk in flight) ----
  {
    const int c4 = kp / 4;
    for (int e = tid; e < nr * c4; e += kNtThreads) {
      const int row = e / c4, c = e % c4;
      const int64_t goff = (int64_t)rows_s[row] * kp + 4 * c;
      cp_async16(V + (size_t)row * kp + 4 * c, P.D + goff);
      cp_async16(Dn + (size_t)row * kp + 4 * c, P.Bbar + goff);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  if (wid == 0) {
    double dm = 1.0;
    for (int j = lane; j < k; j += 32) dm = fmax(dm, diag_s[j]);
    dm = warp_max(dm);
    if (lane == 0) dmax_s = dm;
  }
  __syncthreads();
  const double dmax = dmax_s;
  for (int p = tid; p < KPT; p += kNtThreads) {
    if (p < k) {
      const int j = jmap_s[p];
      pinv_s[j] = p;
      const double cjj = diag_s[j];
      const bool dead = !(cjj > 1e-12 * dmax);                      // R10
      invc_s[p] = dead ? 0.f : (float)(1.0 / cjj);
      vlo_s[p] = (P.pos && !dead) ? 0.f : -INFINITY;      // D >= 0 clamp; dead atoms keep d
      const double lw = dead ? 0.0 : lws_s[j];
      lam_s[p] = lw;
      rho_s[p] = ns_s[j];         // n_{t-1}^(j); becomes rho_j after round 0
      mode_s[p] = dead ? kModeDead : (lw > 0.0 ? kModeShrink : kModeCopy);
      thf_s[p] = (float)(a * lw);
      scf_s[p] = (float)(1.0 / (1.0 + b * lw));
    } else {
      invc_s[p] = 0.f;
      vlo_s[p] = -INFINITY;
      thf_s[p] = 0.f;
      scf_s[p] = 1.f;
      mode_s[p] = kModeDead;
      lam_s[p] = 0.0;
    }
  }
  asm volatile("cp.async.wait_group 1;" ::: "memory");     // Cbar staged
  __syncthreads();
  for (int e = tid; e < k * KPT; e += kNtThreads) {
    const int p = e / KPT, l = e % KPT;
    const int64_t src = (int64_t)jmap_s[p] * k + (l < k ? jmap_s[l] : 0);
    Cpi[e] = l < k ? (cstage ? Rini[src] : __ldg(P.C32 + src)) : 0.f;
  }
  NT_MARK(76);
  asm volatile("cp.async.wait_group 0;" ::: "memory");     // rows staged
  __syncthreads();
  NT_MARK(77);
  for (int e = tid; e < nr * KPT; e += kNtThreads) {
    const int row = e / KPT, p = e % KPT;
    const bool in = p < k;
    const int j = in ? jmap_s[p] : 0;
    Dold[(size_t)row * LD + p] = in ? V[(size_t)row * kp + j] : 0.f;
    Rini[(size_t)row * LD + p] = in ? Dn[(size_t)row * kp + j] : 0.f;
  }
  __syncthreads();
  NT_MARK(78);
  // R = P Bbar - P D Cbar: 8 rows x 8 positions per item (about one item per thread)
  {
    const int nrb = (nr + 7) / 8, npb = (k + 7) / 8;
    for (int it = tid; it < nrb * npb; it += kNtThreads) {
      const int r0 = (it / npb) * 8, p0 = (it % npb) * 8;
      float acc[8][8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[i][c] = 0.f;
      for (int l = 0; l < k; ++l) {
        const float4 c0 = *reinterpret_cast<const float4*>(Cpi + (size_t)l * KPT + p0);
        const float4 c1 = *reinterpret_cast<const float4*>(Cpi + (size_t)l * KPT + p0 + 4);
        const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float d = Dold[(size_t)min(r0 + i, cap - 1) * LD + l];
#pragma unroll
          for (int c = 0; c < 8; ++c) acc[i][c] = fmaf(d, cv[c], acc[i][c]);
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int row = r0 + i;
        if (row >= nr) continue;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int p = p0 + c;
          if (p < k) Rini[(size_t)row * LD + p] -= acc[i][c];
        }
      }
    }
  }
  __syncthreads();

  // stats partial layout: H groups of threads per atom
  const int H = max(1, kNtThreads / max(k, 1));
  double* pc = part;                              // [H][KPT] count
  double* p1 = pc + H * KPT;                      // [H][KPT] S1
  double* p2 = p1 + H * KPT;                      // [H][KPT] S2
  unsigned* pmn = reinterpret_cast<unsigned*>(p2 + H * KPT);   // [H][KPT]
  unsigned* pmx = pmn + H * KPT;                                // [H][KPT]

  NT_MARK(0);
  unsigned nbar = 0;
  int round = 0;
  bool done = q == 0;
  while (!done) {
    // ---- 1. the recurrence, thread per row ------------------------------------
    if (tid < nr) {
      const int row = tid;
      float R[KPT];
#pragma unroll
      for (int p = 0; p < KPT; ++p) R[p] = Rini[(size_t)row * LD + p];
      NtRec<KPT, 0>::run(R, Dold + (size_t)row * LD, V + (size_t)row * LD, Dn + (size_t)row * LD, Cpi, invc_s,
                         thf_s, scf_s, vlo_s, k);
    }
    __syncthreads();
    NT_MARK(1);
    // ---- 2. per-atom statistics over my rows, then one grid reduction -----------
    const int ring = round % kNtRing;
    if (tid < H * k) {
      const int p = tid % k, h = tid / k;
      const double th = a * lam_s[p];
      const bool thr_zero = !(th > 0.0);
      // fp32 partials over <= cap/H rows (relative error ~1e-6),
      // fp64 from here on.  The test is exact: for a float |v| and a double
      // th, |v| > th  <=>  |v| > round_down_to_float(th).
      int cnt = 0;
      float s1 = 0.f, s2 = 0.f;
      unsigned mn = 0xffffffffu, mx = 0u;
      const float thf = thr_zero ? 0.f : __double2float_rd(th);
#pragma unroll 4
      for (int row = h; row < nr; row += H) {
        const float av = fabsf(V[(size_t)row * LD + p]);
        if (av > thf) {
          ++cnt;
          s1 += av;
          s2 = fmaf(av, av, s2);
          mn = min(mn, __float_as_uint(av));
        } else {
          mx = max(mx, __float_as_uint(av));
        }
      }
      pc[h * KPT + p] = (double)cnt;
      p1[h * KPT + p] = (double)s1;
      p2[h * KPT + p] = (double)s2;
      pmn[h * KPT + p] = mn;
      pmx[h * KPT + p] = mx;
    }
    __syncthreads();
    if (tid < k) {
      const int p = tid;
      double cnt = 0.0, s1 = 0.0, s2 = 0.0;
      unsigned mn = 0xffffffffu, mx = 0u;
      for (int h = 0; h < H; ++h) {
        cnt += pc[h * KPT + p];
        s1 += p1[h * KPT + p];
        s2 += p2[h * KPT + p];
        mn = min(mn, pmn[h * KPT + p]);
        mx = max(mx, pmx[h * KPT + p]);
      }
      double* acc = P.acc + ((size_t)ring * k + p) * 3;
      unsigned* mm = P.accmm + ((size_t)ring * k + p) * 2;
      if (nr > 0) {
        if (cnt > 0.0) {
          nt_red_add(acc, cnt);
          nt_red_add(acc + 1, s1);
          nt_red_add(acc + 2, s2);
          atomicMin(mm, mn);
        }
        if (mx) atomicMax(mm + 1, mx);
        if (round == 0) {
          // radii (R9): ||P d_j|| of the column before its update
          double d1 = 0.0, d2 = 0.0;
          for (int row = 0; row < nr; ++row) {
            const double d = Dold[(size_t)row * LD + p];
            d1 += fabs(d);
            d2 += d * d;
          }
          nt_red_add(P.rho_acc + 2 * p, d1);
          nt_red_add(P.rho_acc + 2 * p + 1, d2);
        }
      }
    }
    NT_MARK(2);
    ++nbar;
    nt_barrier(P.bar, nbar * G);
    NT_MARK(3);
    if (blockIdx.x == 0) {
      // recycle the ring slot of the NEXT-but-one round (its readers are done)
      const int rz = (round + 2) % kNtRing;
      for (int e = tid; e < 3 * k; e += kNtThreads) P.acc[(size_t)rz * k * 3 + e] = 0.0;
      for (int e = tid; e < k; e += kNtThreads) {
        P.accmm[((size_t)rz * k + e) * 2] = 0xffffffffu;
        P.accmm[((size_t)rz * k + e) * 2 + 1] = 0u;
      }
    }
    // ---- 3. the same Michelot step for every atom in every CTA -----------------
    int conv = 1;
    if (tid < k) {
      const int p = tid;
      if (round == 0) {
        const double d1 = __ldcg(P.rho_acc + 2 * p), d2 = __ldcg(P.rho_acc + 2 * p + 1);
        rho_s[p] = fmax(0.0, rho_s[p] + a * d1 + 0.5 * b * d2);          // P:860, R9
      }
      const double rho = rho_s[p];
      const double* acc = P.acc + ((size_t)ring * k + p) * 3;
      const unsigned* mm = P.accmm + ((size_t)ring * k + p) * 2;
      const double cnt = __ldcg(acc), S1 = __ldcg(acc + 1), S2 = __ldcg(acc + 2);
      const double mnv = cnt > 0.0 ? (double)__uint_as_float(__ldcg(mm)) : INFINITY;
      const double mxv = (double)__uint_as_float(__ldcg(mm + 1));
      const int mode = mode_s[p];
      const double lam = lam_s[p];
      int nmode;
      double nlam;
      conv = nt_atom_update(a, b, rho, cnt, S1, S2, mnv, mxv, mode, lam, &nmode, &nlam);
      lam_s[p] = nlam;
      mode_s[p] = nmode;
      thf_s[p] = nmode == kModeShrink ? (float)(a * nlam) : 0.f;
      scf_s[p] = nmode == kModeShrink ? (float)(1.0 / (1.0 + b * nlam)) : nmode == kModeZero ? 0.f : 1.f;
    }
    const int all = __syncthreads_and(conv);
    if (P.prof && blockIdx.x == 0) {
      // convergence profile: unconverged atoms per round (slots 8..71)
      const int nun = __syncthreads_count(!conv);
      if (tid == 0 && round < 64) P.prof[8 + round] += nun;
    }
    NT_MARK(4);
    ++round;
    if (all) {
      done = true;
    } else if (round >= P.max_rounds) {
      if (tid == 0 && blockIdx.x == 0) atomicExch(P.err, 4);
      done = true;
    }
    if (done && tid < k) {
      // slack n_j = rho_j - ||d_j|| from the sums of this (final) round
      const int p = tid, j = jmap_s[p];
      const int mode = mode_s[p];
      if (mode != kModeDead && blockIdx.x == 0) {
        const double* acc = P.acc + ((size_t)ring * k + p) * 3;
        const double cnt = __ldcg(acc), S1 = __ldcg(acc + 1), S2 = __ldcg(acc + 2);
        const double Nd = nt_norm_d(a, b, mode, lam_s[p], cnt, S1, S2);
        P.nslack[j] = rho_s[p] - Nd;
        P.lam_ws[j] = lam_s[p];
      }
    }
  }
  __syncthreads();
  NT_MARK(5);
  // ---- final D = the last round's d (what its recurrence used), in atom order ------
  if (q > 0) {
    for (int row = wid; row < nr; row += kNtThreads / 32) {
      float* dst = P.D + (int64_t)rows_s[row] * kp;
      const float* src = Dn + (size_t)row * LD;
      for (int j = lane; j < k; j += 32) dst[j] = src[pinv_s[j]];
    }
  }
  // ---- exit: last CTA resets counters and accumulators ------------------------------
  __syncthreads();
  NT_MARK(6);
  if (P.prof && blockIdx.x == 0 && threadIdx.x == 0) P.prof[7] += 1;
  if (tid == 0) {
    __threadfence();
    const unsigned old = atomicAdd(P.bar + 1, 1u);
    if (old == (unsigned)G - 1) {
      __threadfence();
      for (int e = 0; e < kNtRing * k * 3; ++e) P.acc[e] = 0.0;
      for (int e = 0; e < kNtRing * k; ++e) {
        P.accmm[2 * e] = 0xffffffffu;
        P.accmm[2 * e + 1] = 0u;
      }
      for (int e = 0; e < 2 * k; ++e) P.rho_acc[e] = 0.0;
      if (P.nred_out) *P.nred_out = nbar;
      P.bar[0] = 0u;
      P.bar[1] = 0u;
      __threadfence();
    }
  }
}

}  // namespace somf
