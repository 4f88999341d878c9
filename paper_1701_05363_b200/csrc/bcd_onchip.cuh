// bcd_onchip.cuh -- (a4) partial dictionary update, Alg. 4, v2:
// the q masked rows stay on chip for the whole pass.
//
// One persistent cooperative kernel, one 512-thread CTA per SM.  CTA b owns
// the masked rows [q b / G, q (b+1) / G) of the index list.  Per row it keeps
//   * D_M row          in shared memory (Dm, k padded to kp),
//   * the residual     R = P_t Bbar - P_t D Cbar   in REGISTERS, one warp per
//                      row, lane l holding columns l, l+32, ... (KC per lane).
// Alg. 4's update of atom j reads only column j of R:
//   u_i = d_ij + R_ij / Cbar_jj ,
// and after the projection the new column changes R by a rank-1 term
//   R_i: -= (d_ij^new - d_ij) Cbar_j:          (k FMAs per row, no reduction)
// so each atom costs O(k) per row and no re-read of D_M (the oracle's
// "D[S,:] Cbar[:,j]" with D[S,:] holding the atoms already updated).
//
// Radii (R9): rho_j = n_j + ||P d_j|| depends only on column j before
// its own update, so all k radii come from ONE grid reduction before the pass.
//
// Projection threshold (R17), sort-free and exact:
//   every round reduces, over the grid, for NC candidate thresholds th_c the
//   sums (count, S1, S2) of the |v_i| > th_c and the smallest such |v_i|
//   (fixed-point u64 red.add / u32 atomicMin into a ring of L2 accumulators, then one
//   grid barrier).  Every CTA then evaluates the same decision:
//     - feasible (||v|| <= rho): lambda = 0;  rho = 0: d = 0;  mu = 1: closed form;
//     - candidate c is a lower bound iff phi(th_c) = ||shrink(v, th_c)|| >= rho;
//       its active-set root lam_c (enet_lambda) is EXACT iff a lam_c is below
//       the smallest active |v| (then {|v| > a lam_c} is the same set);
//     - otherwise L = max a lam_c over lower bounds (a Michelot step, so the
//       iteration never does worse than Michelot's) and U = min upper bound
//       th_c; the next round probes L and NC-1 points in (L, U).
//   Round 1 probes 0 (all nonzeros, feasibility) and a fan around the atom's
//   threshold of the previous iteration (warm start).
// All CTAs read identical reduced values, so they take identical decisions.
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kOcThreads = 512;
constexpr int kOcWarps = kOcThreads / 32;
constexpr int kNC = 16;            // candidate thresholds per round (one warp each)
constexpr int kRing = 4;           // accumulator ring (rounds)
constexpr int kMaxRounds = 200;    // safety cap per atom (Michelot terminates far earlier)

struct OcArgs {
  const int32_t* idx;       // masked local rows (ascending)
  const int64_t* q_dev;
  float* D;                 // rows x kp
  const float* Bbar;        // rows x kp
  const double* C64;        // k x k
  const float* C32;         // k x k
  double* nslack;           // k
  double* theta_ws;         // k: a*lambda of the previous pass (warm start)
  const int32_t* perm;      // k
  int k, kp;
  double a, b;              // 1 - mu, mu
  int pos;                  // D >= 0
  int cs_smem;              // Cbar (fp32) staged in shared memory
  int cap_rows;             // rows per CTA the shared memory holds
  unsigned long long* acc;  // [kRing][kNC][5]: count, S1 limbs, S2 limbs (fx_red; zero between uses)
  unsigned* accmin;         // [kRing][kNC]      (0xffffffff between uses)
  unsigned long long* rho_acc;  // [4k]: sum|d_j| limbs, sum d_j^2 limbs (zero between uses)
  unsigned* bar;            // [0] arrivals [1] exits [2] watchdog
  int64_t* nred_out;        // grid reductions performed (diagnostic)
  int* err;                 // 2: more masked rows than capacity
};

// ---------------------------------------------------------------------------
// grid barrier on a monotonic arrival counter (reset by the last CTA to exit)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void oc_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    if (ld_acquire_gpu(bar) < target) {
      const uint64_t t0 = globaltimer_ns();
      unsigned spins = 0;
      while (ld_acquire_gpu(bar) < target) {
        if ((++spins & 1023u) == 0) {
          if (ld_acquire_gpu(bar + 2)) break;                      // watchdog already fired
          if (globaltimer_ns() - t0 > 2000000000ull) { atomicExch(bar + 2, 1u); break; }
        }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// ||shrink(v, th)|| from the sums over {|v| > th}: lam = th / a.
__device__ __forceinline__ double enet_phi(double a, double b, double th, double cnt, double S1,
                                           double S2) {
  const double lam = a > 0.0 ? th / a : 0.0;
  const double opb = 1.0 + b * lam;
  const double s1 = (S1 - cnt * th) / opb;
  const double s2 = (S2 - 2.0 * th * S1 + cnt * th * th) / (opb * opb);
  return a * s1 + 0.5 * b * s2;
}

template <int KC>
__device__ __forceinline__ float pick(const float (&r)[KC], int c) {
  float x = 0.f;
#pragma unroll
  for (int i = 0; i < KC; ++i)
    if (i == c) x = r[i];
  return x;
}

template <int KC, int RPW>
__global__ void __launch_bounds__(kOcThreads, 1)
k_bcd_onchip(OcArgs P) {
  extern __shared__ __align__(16) float oc_smem[];
  __shared__ double thr_s[kNC];
  __shared__ double dec_s[8];        // lam, rho, Nd, mode
  __shared__ int done_s;
  __shared__ double dmax_s;
  const int k = P.k, kp = P.kp;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int64_t q = *P.q_dev;
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  int nr = (int)(hi - lo);
  if (nr > P.cap_rows || nr > RPW * kOcWarps) {
    if (tid == 0) atomicExch(P.err, 2);
    nr = min(P.cap_rows, RPW * kOcWarps);
  }
  float* Dm = oc_smem;                                   // cap_rows x kp
  float* Cs = Dm + (size_t)P.cap_rows * kp;              // k x k (if cs_smem)
  float* vbuf = Cs + (P.cs_smem ? (size_t)((k * k + 3) & ~3) : 0);   // cap_rows
  double* rho_s = reinterpret_cast<double*>(vbuf + ((P.cap_rows + 1) & ~1));   // k
  double* ws_s = rho_s + k;                               // k
  int* perm_s = reinterpret_cast<int*>(ws_s + k);         // k
  const double a = P.a, b = P.b;

  // ---- stage rows, Cbar, perm, warm starts -------------------------------
  for (int row = wid; row < nr; row += kOcWarps) {
    const float4* src = reinterpret_cast<const float4*>(P.D + (int64_t)P.idx[lo + row] * kp);
    float4* dst = reinterpret_cast<float4*>(Dm + (size_t)row * kp);
    for (int c = lane; c < kp / 4; c += 32) dst[c] = src[c];
  }
  if (P.cs_smem)
    for (int e = tid; e < k * k; e += kOcThreads) Cs[e] = P.C32[e];
  for (int j = tid; j < k; j += kOcThreads) {
    perm_s[j] = P.perm[j];
    ws_s[j] = P.theta_ws[j];
  }
  if (tid == 0) {
    double dm = 1.0;
    for (int j = 0; j < k; ++j) dm = fmax(dm, P.C64[(int64_t)j * k + j]);
    dmax_s = dm;
  }
  __syncthreads();

  // ---- radii: one grid reduction of (sum|d_j|, sum d_j^2) over the masked rows
  for (int j = tid; j < k; j += kOcThreads) {
    double s1 = 0.0, s2 = 0.0;
    for (int row = 0; row < nr; ++row) {
      const double d = Dm[(size_t)row * kp + j];
      s1 += fabs(d);
      s2 += d * d;
    }
    if (nr > 0) {
      if (!(fx_red(P.rho_acc + 4 * j, s1) & fx_red(P.rho_acc + 4 * j + 2, s2))) atomicExch(P.err, 6);
    }
  }
  // ---- residual R = Bbar_M - D_M Cbar (registers) --------------------------
  float R[RPW][KC];
#pragma unroll
  for (int s = 0; s < RPW; ++s) {
    const int row = wid + kOcWarps * s;
    const int64_t g = row < nr ? (int64_t)P.idx[lo + row] : 0;
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const int col = lane + 32 * c;
      R[s][c] = (row < nr && col < k) ? P.Bbar[g * kp + col] : 0.f;
    }
  }
  for (int l = 0; l < k; ++l) {
    float cl[KC];
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      const int col = lane + 32 * c;
      cl[c] = col < k ? (P.cs_smem ? Cs[l * k + col] : __ldg(P.C32 + (int64_t)l * k + col)) : 0.f;
    }
#pragma unroll
    for (int s = 0; s < RPW; ++s) {
      const int row = wid + kOcWarps * s;
      const float d = row < nr ? Dm[(size_t)row * kp + l] : 0.f;
#pragma unroll
      for (int c = 0; c < KC; ++c) R[s][c] = fmaf(-d, cl[c], R[s][c]);
    }
  }
  unsigned nbar = 1;
  oc_barrier(P.bar, nbar * G);
  for (int j = tid; j < k; j += kOcThreads) {
    const double s1 = fx_value(__ldcg(P.rho_acc + 4 * j), __ldcg(P.rho_acc + 4 * j + 1));
    const double s2 = fx_value(__ldcg(P.rho_acc + 4 * j + 2), __ldcg(P.rho_acc + 4 * j + 3));
    rho_s[j] = fmax(0.0, P.nslack[j] + a * s1 + 0.5 * b * s2);       // P:860, R9
  }
  __syncthreads();
  const double dmax = dmax_s;
  int ring = 0;

  // ---- Alg. 4: atoms in permutation order -----------------------------------
  if (q > 0) {
    for (int pi = 0; pi < k; ++pi) {
      const int j = perm_s[pi];
      const double cjj = P.C64[(int64_t)j * k + j];
      if (!(cjj > 1e-12 * dmax)) continue;                      // R10: dead atom
      const float invc = (float)(1.0 / cjj);
      const int ol = j & 31, cj = j >> 5;
      // column j of R of my warp's rows -> lanes 0..RPW-1
      float myr = 0.f;
#pragma unroll
      for (int s = 0; s < RPW; ++s) {
        const float x = __shfl_sync(0xffffffffu, pick<KC>(R[s], cj), ol);
        if (lane == s) myr = x;
      }
      const int myrow = wid + kOcWarps * lane;
      const bool own = lane < RPW && myrow < nr;
      float myd = 0.f, myv = 0.f;
      if (own) {
        myd = Dm[(size_t)myrow * kp + j];
        const float u = fmaf(myr, invc, myd);
        myv = P.pos ? fmaxf(u, 0.f) : u;
        vbuf[myrow] = myv;
      }
      float cjv[KC];
#pragma unroll
      for (int c = 0; c < KC; ++c) {
        const int col = lane + 32 * c;
        cjv[c] = col < k ? (P.cs_smem ? Cs[j * k + col] : __ldg(P.C32 + (int64_t)j * k + col)) : 0.f;
      }
      const double rho = rho_s[j];
      if (tid < kNC) {
        // round-1 probes: 0 (every nonzero) and a fan around the warm start
        const double w0 = ws_s[j];
        double th = 0.0;
        if (tid > 0 && w0 > 0.0) {
          // factors 1 -+ 0.001 * 3^(|s|-1), s = -7..7 (0.27 .. 1.73)
          const int sm = tid - 8;
          double f = 0.0;
          if (sm != 0) {
            f = 0.001;
            for (int e = 1; e < abs(sm); ++e) f *= 3.0;
          }
          th = w0 * (sm < 0 ? 1.0 - f : 1.0 + f);
        }
        thr_s[tid] = th;
      }
      if (tid == 0) done_s = 0;
      __syncthreads();
      int round = 0;
      while (true) {
        // candidate partial sums: warp w -> threshold w
        if (wid < kNC) {
          const double th = thr_s[wid];
          double cnt = 0.0, s1 = 0.0, s2 = 0.0;
          unsigned mn = 0xffffffffu;
          for (int row = lane; row < nr; row += 32) {
            const float v = vbuf[row];
            const double av = fabs((double)v);
            if (av > th) {
              cnt += 1.0;
              s1 += av;
              s2 += av * av;
              mn = min(mn, __float_as_uint(fabsf(v)));
            }
          }
          cnt = warp_sum(cnt);
          s1 = warp_sum(s1);
          s2 = warp_sum(s2);
          mn = __reduce_min_sync(0xffffffffu, mn);
          if (lane == 0 && cnt > 0.0) {
            unsigned long long* acc = P.acc + ((size_t)ring * kNC + wid) * 5;
            nt_red_u64(acc, (unsigned long long)cnt);
            if (!(fx_red(acc + 1, s1) & fx_red(acc + 3, s2))) atomicExch(P.err, 6);
            atomicMin(P.accmin + ring * kNC + wid, mn);
          }
        }
        ++nbar;
        oc_barrier(P.bar, nbar * G);
        if (blockIdx.x == 0 && tid < kNC * 4) {
          // recycle the ring slot two rounds ahead (its last readers are done)
          const int rz = (ring + 2) % kRing;
          if (tid < kNC * 3) {
            unsigned long long* z = P.acc + ((size_t)rz * kNC + tid / 3) * 5;
            if (tid % 3 == 0) z[0] = 0ull;
            else if (tid % 3 == 1) { z[1] = 0ull; z[2] = 0ull; }
            else { z[3] = 0ull; z[4] = 0ull; }
          } else {
            P.accmin[rz * kNC + (tid - kNC * 3)] = 0xffffffffu;
          }
        }
        if (wid == 0) {
          const int c = lane;
          double cnt = 0.0, S1 = 0.0, S2 = 0.0, th = 0.0, mnv = 0.0;
          if (c < kNC) {
            const unsigned long long* acc = P.acc + ((size_t)ring * kNC + c) * 5;
            cnt = (double)__ldcg(acc);
            S1 = fx_value(__ldcg(acc + 1), __ldcg(acc + 2));
            S2 = fx_value(__ldcg(acc + 3), __ldcg(acc + 4));
            mnv = (double)__uint_as_float(__ldcg(P.accmin + ring * kNC + c));
            th = thr_s[c];
          }
          // lane 0: in round 0 probe 0 = every nonzero -> feasibility / closed forms
          const double Nv0 = __shfl_sync(0xffffffffu, a * S1 + 0.5 * b * S2, 0);
          const double cnt0 = __shfl_sync(0xffffffffu, cnt, 0);
          const double S10 = __shfl_sync(0xffffffffu, S1, 0);
          const double S20 = __shfl_sync(0xffffffffu, S2, 0);
          int mode = -1;          // 0: copy v, 1: zero, 2: shrink with lam
          double lam = 0.0, Nd = 0.0;
          if (round == 0 && Nv0 <= rho) { mode = 0; Nd = Nv0; }
          else if (round == 0 && !(rho > 0.0)) { mode = 1; Nd = 0.0; }
          else if (round == 0 && !(a > 0.0)) {
            mode = 2;
            lam = enet_lambda(a, b, rho, cnt0, S10, S20);
            const double opb = 1.0 + b * lam;
            Nd = 0.5 * b * S20 / (opb * opb);
          } else {
            bool valid = false, exact = false;
            double lamc = 0.0, phic = 0.0;
            if (c < kNC && cnt > 0.0) {
              phic = enet_phi(a, b, th, cnt, S1, S2);
              // probe 0 of a later round is the previous Michelot iterate: a
              // lower bound by construction (rounding must not demote it)
              valid = phic >= rho || (c == 0 && round > 0);
              if (valid) {
                lamc = enet_lambda(a, b, rho, cnt, S1, S2);
                exact = a * lamc < mnv;
              }
            }
            const unsigned ex = __ballot_sync(0xffffffffu, exact);
            if (ex) {
              const int src = __ffs(ex) - 1;
              lam = __shfl_sync(0xffffffffu, lamc, src);
              const double sc = __shfl_sync(0xffffffffu, cnt, src);
              const double s1 = __shfl_sync(0xffffffffu, S1, src);
              const double s2 = __shfl_sync(0xffffffffu, S2, src);
              const double t = a * lam, opb = 1.0 + b * lam;
              Nd = a * (s1 - sc * t) / opb + 0.5 * b * (s2 - 2.0 * t * s1 + sc * t * t) / (opb * opb);
              mode = 2;
            } else {
              double L = valid ? a * lamc : 0.0;
              double U = (c < kNC && !valid) ? th : INFINITY;
              L = warp_max(L);
              if (round > 0) L = fmax(L, __shfl_sync(0xffffffffu, th, 0));
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) U = fmin(U, __shfl_xor_sync(0xffffffffu, U, o));
              if (round + 1 >= kMaxRounds) {
                // safety net (not expected): Michelot iterate as the answer
                mode = 2;
                lam = L / a;
                Nd = rho;
                if (lane == 0 && blockIdx.x == 0) atomicExch(P.err, 3);
              } else if (c < kNC) {
                double nt;
                if (c == 0) nt = L;
                else if (U < INFINITY && U > L) nt = L + (U - L) * ((double)c / kNC);
                else nt = L * (1.0 + 0.002 * c * c);
                thr_s[c] = nt;
              }
            }
          }
          if (lane == 0 && mode >= 0) {
            dec_s[0] = lam;
            dec_s[1] = Nd;
            dec_s[2] = (double)mode;
            done_s = 1;
          }
        }
        __syncthreads();
        ring = (ring + 1) % kRing;
        ++round;
        if (done_s) break;
      }
      // ---- apply: d_j on my rows, rank-1 update of R -------------------------
      const double lam = dec_s[0];
      const int mode = (int)dec_s[2];
      float delta = 0.f;
      if (own) {
        float d;
        if (mode == 0) d = myv;
        else if (mode == 1) d = 0.f;
        else d = copysignf((float)(fmax(fabs((double)myv) - a * lam, 0.0) / (1.0 + b * lam)), myv);
        Dm[(size_t)myrow * kp + j] = d;
        delta = d - myd;
      }
#pragma unroll
      for (int s = 0; s < RPW; ++s) {
        const float dl = __shfl_sync(0xffffffffu, delta, s);
        if (dl != 0.f) {
#pragma unroll
          for (int c = 0; c < KC; ++c) R[s][c] = fmaf(-dl, cjv[c], R[s][c]);
        }
      }
      if (blockIdx.x == 0 && tid == 0) {
        P.nslack[j] = rho - dec_s[1];
        P.theta_ws[j] = mode == 2 ? a * lam : P.theta_ws[j];
      }
      __syncthreads();
    }
  }
  // ---- write D_M back (rows outside S_t untouched: freezing) ----
  for (int row = wid; row < nr; row += kOcWarps) {
    float4* dst = reinterpret_cast<float4*>(P.D + (int64_t)P.idx[lo + row] * kp);
    const float4* src = reinterpret_cast<const float4*>(Dm + (size_t)row * kp);
    for (int c = lane; c < kp / 4; c += 32) dst[c] = src[c];
  }
  // ---- exit: the last CTA resets the counters and the accumulators ---------
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned old = atomicAdd(P.bar + 1, 1u);
    if (old == (unsigned)G - 1) {
      __threadfence();
      for (int e = 0; e < kRing * kNC * 5; ++e) P.acc[e] = 0ull;
      for (int e = 0; e < kRing * kNC; ++e) P.accmin[e] = 0xffffffffu;
      for (int e = 0; e < 4 * k; ++e) P.rho_acc[e] = 0ull;
      if (P.nred_out) *P.nred_out = nbar;
      P.bar[0] = 0u;
      P.bar[1] = 0u;
      __threadfence();
    }
  }
}

}  // namespace somf
