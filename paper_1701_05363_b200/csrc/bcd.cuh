// bcd.cuh -- (a4) partial dictionary update, Alg. 4, and the
// elastic-net ball projection it calls.
//
// v1 (this file): atoms strictly in Alg. 4's order, one cooperative kernel.
// Each CTA owns a contiguous slice of the q masked rows; per atom j:
//   u_i = d_ij + (bbar_ij - sum_l d_il cbar_lj) / cbar_jj
//   one grid reduction -> ||P d_j|| (radius) and ||v|| (feasibility)
//   if infeasible: sort-free active-set (Michelot) iterations, one grid
//   reduction of (count, S1, S2) each, lambda from the active-set quadratic
//   d_i = sign(v_i) max(|v_i| - a lam, 0) / (1 + b lam)             (R17)
//   n_j = rho - ||d_j|| from the same sums
// Reductions are fixed-order (per-CTA partials, then the same tree in every
// CTA), so all CTAs agree bit-for-bit on rho, lambda and n_j.
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kBcdThreads = 256;
constexpr int kRedStride = 8;     // doubles per CTA partial slot

struct BcdArgs {
  const int32_t* idx;       // masked local rows (ascending), or nullptr = rows 0..q-1
  const int64_t* q_dev;
  float* D;                 // rows x kp
  const float* Bbar;        // rows x kp
  const double* C64;        // k x k
  const float* C32;         // k x k
  double* nslack;           // k
  const int32_t* perm;      // k
  int k, kp;
  double a, b;              // 1 - mu, mu
  int pos;                  // D >= 0
  double* red;              // [2][gridDim][kRedStride]
  unsigned* bar;            // grid barrier {count, generation}
  int64_t* nred_out;        // reductions performed (diagnostic)
};

// Fixed-order grid reduction of N (<= kRedStride) doubles.
template <int N>
__device__ __forceinline__ void grid_reduce(double (&v)[N], double* red, unsigned* bar, int& parity,
                                            double* scratch, double* bcast) {
  block_sum<N>(v, scratch);
  const int G = gridDim.x;
  double* slot = red + ((size_t)parity * G + blockIdx.x) * kRedStride;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) slot[i] = v[i];
  }
  grid_barrier(bar);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0;
      for (int b = lane; b < G; b += 32) s += __ldcg(red + ((size_t)parity * G + b) * kRedStride + i);
      s = warp_sum(s);
      if (lane == 0) bcast[i] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = bcast[i];
  __syncthreads();
  parity ^= 1;
}

// smem: k floats (column of Cbar) + rows_cap floats (v of owned rows)
__global__ void __launch_bounds__(kBcdThreads)
k_bcd_seq(BcdArgs P) {
  extern __shared__ float smf[];
  __shared__ double scratch[kRedStride * 32];
  __shared__ double bcast[kRedStride];
  __shared__ double dmax_s;
  float* ccol = smf;
  float* vbuf = smf + ((P.k + 3) & ~3);
  const int k = P.k, kp = P.kp, tid = threadIdx.x, nt = blockDim.x;
  const int64_t q = *P.q_dev;
  const int G = gridDim.x;
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  const double a = P.a, b = P.b;
  int parity = 0;
  int64_t nred = 0;
  if (tid == 0) {
    double dm = 1.0;
    for (int j = 0; j < k; ++j) dm = fmax(dm, P.C64[(int64_t)j * k + j]);
    dmax_s = dm;
  }
  __syncthreads();
  const double dmax = dmax_s;
  for (int pi = 0; pi < k; ++pi) {
    const int j = P.perm[pi];
    const double cjj = P.C64[(int64_t)j * k + j];
    if (!(cjj > 1e-12 * dmax)) continue;                       // R10: dead atom
    // n_j is read before this atom's first grid barrier: block 0 rewrites it
    // after the atom's last barrier, so every CTA sees the same n_{t-1}^(j).
    const double nj = P.nslack[j];
    for (int l = tid; l < k; l += nt) ccol[l] = P.C32[(int64_t)j * k + l];
    __syncthreads();
    const float invc = (float)(1.0 / cjj);
    double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};   // |d|, d^2, #v!=0, |v|, v^2
    for (int64_t m = lo + tid; m < hi; m += nt) {
      const int64_t g = P.idx ? (int64_t)P.idx[m] : m;
      const float* row = P.D + g * kp;
      float dot = 0.f;
      for (int l = 0; l < k; ++l) dot = fmaf(row[l], ccol[l], dot);
      const float dj = row[j];
      const float u = fmaf(P.Bbar[g * kp + j] - dot, invc, dj);
      const float v = P.pos ? fmaxf(u, 0.f) : u;
      vbuf[m - lo] = v;
      s[0] += fabs((double)dj);
      s[1] += (double)dj * dj;
      s[2] += v != 0.f ? 1.0 : 0.0;
      s[3] += fabs((double)v);
      s[4] += (double)v * v;
    }
    grid_reduce<5>(s, P.red, P.bar, parity, scratch, bcast);
    ++nred;
    const double rho = fmax(0.0, nj + a * s[0] + 0.5 * b * s[1]);            // P:860, R9
    const double Nv = a * s[3] + 0.5 * b * s[4];
    double lam = 0.0, Nd = Nv;
    bool zero = false;
    if (Nv > rho) {
      if (!(rho > 0.0)) { zero = true; Nd = 0.0; }                       // R11
      else {
        double cnt = s[2], S1 = s[3], S2 = s[4];
        lam = enet_lambda(a, b, rho, cnt, S1, S2);
        if (a > 0.0) {
          // Michelot: shrink the active set {|v| > a lam} until it is stable
          // (threshold compared in float64: a float-rounded a*lam can exclude
          // the last active entry and make the iteration cycle)
          for (int it = 0; it < 4096; ++it) {
            const double thr = a * lam;
            double t3[3] = {0.0, 0.0, 0.0};
            for (int64_t m = lo + tid; m < hi; m += nt) {
              const float v = vbuf[m - lo];
              const double av = fabs((double)v);
              if (av > thr) { t3[0] += 1.0; t3[1] += av; t3[2] += av * av; }
            }
            grid_reduce<3>(t3, P.red, P.bar, parity, scratch, bcast);
            ++nred;
            if (t3[0] == cnt || t3[0] == 0.0) break;
            cnt = t3[0]; S1 = t3[1]; S2 = t3[2];
            lam = enet_lambda(a, b, rho, cnt, S1, S2);
          }
        }
        const double opb = 1.0 + b * lam;
        const double sd = (S1 - cnt * a * lam) / opb;
        const double sd2 = (S2 - 2.0 * a * lam * S1 + cnt * a * a * lam * lam) / (opb * opb);
        Nd = a * sd + 0.5 * b * sd2;
      }
    }
    const double thr = a * lam;
    const double inv1 = 1.0 / (1.0 + b * lam);
    for (int64_t m = lo + tid; m < hi; m += nt) {
      const int64_t g = P.idx ? (int64_t)P.idx[m] : m;
      const float v = vbuf[m - lo];
      float d;
      if (zero) d = 0.f;
      else if (lam == 0.0) d = v;
      else d = copysignf((float)(fmax(fabs((double)v) - thr, 0.0) * inv1), v);
      P.D[g * kp + j] = d;
    }
    if (blockIdx.x == 0 && tid == 0) P.nslack[j] = rho - Nd;
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0 && P.nred_out) *P.nred_out = nred;
}

// ---------------------------------------------------------------------------
// One CTA per column: Out[:, j] = Proj(U[:, j]; radius[j], mu, positive);
// optionally nslack[j] = radius[j] - ||Out[:, j]|| (set_components).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kBcdThreads)
k_project_columns(const float* __restrict__ U, int64_t len, int64_t ld, const double* __restrict__ radius,
                  double radius_const, double a, double b, int pos, float* __restrict__ Out,
                  double* __restrict__ nslack) {
  __shared__ double scratch[4 * 32];
  const int j = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const double rho = radius ? radius[j] : radius_const;
  double s[3] = {0.0, 0.0, 0.0};
  for (int64_t i = tid; i < len; i += nt) {
    float v = U[i * ld + j];
    if (pos) v = fmaxf(v, 0.f);
    s[0] += v != 0.f ? 1.0 : 0.0;
    s[1] += fabs((double)v);
    s[2] += (double)v * v;
  }
  block_sum<3>(s, scratch);
  const double Nv = a * s[1] + 0.5 * b * s[2];
  double lam = 0.0;
  bool zero = false;
  if (Nv > rho) {
    if (!(rho > 0.0)) zero = true;
    else {
      double cnt = s[0], S1 = s[1], S2 = s[2];
      lam = enet_lambda(a, b, rho, cnt, S1, S2);
      if (a > 0.0) {
        for (int it = 0; it < 4096; ++it) {
          const double thr = a * lam;
          double t3[3] = {0.0, 0.0, 0.0};
          for (int64_t i = tid; i < len; i += nt) {
            float v = U[i * ld + j];
            if (pos) v = fmaxf(v, 0.f);
            const double av = fabs((double)v);
            if (av > thr) { t3[0] += 1.0; t3[1] += av; t3[2] += av * av; }
          }
          block_sum<3>(t3, scratch);
          if (t3[0] == cnt || t3[0] == 0.0) break;
          cnt = t3[0]; S1 = t3[1]; S2 = t3[2];
          lam = enet_lambda(a, b, rho, cnt, S1, S2);
        }
      }
    }
  }
  __syncthreads();
  const double thr = a * lam;
  const double inv1 = 1.0 / (1.0 + b * lam);
  double nd[2] = {0.0, 0.0};
  for (int64_t i = tid; i < len; i += nt) {
    float v = U[i * ld + j];
    if (pos) v = fmaxf(v, 0.f);
    float d;
    if (zero) d = 0.f;
    else if (lam == 0.0) d = v;
    else d = copysignf((float)(fmax(fabs((double)v) - thr, 0.0) * inv1), v);
    Out[i * ld + j] = d;
    nd[0] += fabs((double)d);
    nd[1] += (double)d * d;
  }
  if (nslack) {
    block_sum<2>(nd, scratch);
    if (tid == 0) nslack[j] = rho - (a * nd[0] + 0.5 * b * nd[1]);
  }
}

}  // namespace somf
