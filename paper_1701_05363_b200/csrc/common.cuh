// common.cuh -- shared device helpers of the SOMF hot path (sm_100a).
//
// Philox4x32-10 (R1), warp/block reductions with a FIXED combination order
// (so every CTA and every run produces the same bits), and a sense-reversing
// grid barrier for cooperative launches.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace somf {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// Philox4x32-10: key = (seed lo, seed hi); counter (c0,c1,c2,c3).
// Draw layout (R1): c2 = stream (1 mask, 2 atom permutation, 3 column ids).
// ---------------------------------------------------------------------------
struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint64_t seed) {
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int rnd = 0; rnd < 10; ++rnd) {
    if (rnd) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

__host__ __device__ __forceinline__ uint32_t u4_word(const U4& v, int lane) {
  return lane == 0 ? v.x : lane == 1 ? v.y : lane == 2 ? v.z : v.w;
}

enum : uint32_t { kStreamMask = 1, kStreamPerm = 2, kStreamCols = 3 };

// Aggregation coefficients of iteration t (Eq. somf_partial, R6),
// kept on the device next to t (w_dev[0..3]) and written by whichever kernel
// begins the iteration (k_step_mask_count or the previous BCD's draw-ahead):
//   Cbar <- keep Cbar + (gc / eta) A A^T ,  P_t Bbar <- keep P_t Bbar + (gb / eta) X_M A^T
// modes M / F: keep = 1 - w_t, gb = gc = w_t.  Mode U stores Bbar / sigma_t and
// Cbar / sigma_t (sigma_t = prod (1 - w_s), the lazy global decay of R6):
// keep = 1, gb = w_t r / sigma_t, gc = w_t / sigma_t.  Alg. 4 is invariant to
// the joint scale of (Bbar, Cbar), so the BCD kernels read the stored values.
enum : int { kCoefW = 0, kCoefKeep = 1, kCoefGainB = 2, kCoefGainC = 3, kCoefN = 4 };
struct StepCoef { double v[kCoefN]; };

__device__ __forceinline__ void store_coef(double* dst, const StepCoef& c) {
#pragma unroll
  for (int i = 0; i < kCoefN; ++i) dst[i] = c.v[i];
}

// Selection bits of the 4 rows of Philox block blk (rows 4 blk .. 4 blk + 3)
// in M_t (Eq. mt; R1, R2): row i selected iff word_{i&3} < T(r).
__device__ __forceinline__ uint32_t mask_bits(uint64_t seed, uint64_t t, int64_t blk,
                                              int64_t row_lo, int64_t row_hi, uint64_t T) {
  const U4 w = philox4x32_10(U4{(uint32_t)blk, (uint32_t)t, kStreamMask, (uint32_t)(blk >> 32)}, seed);
  uint32_t bits = 0;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    const int64_t row = blk * 4 + l;
    if (row >= row_lo && row < row_hi && (uint64_t)u4_word(w, l) < T) bits |= 1u << l;
  }
  return bits;
}

// ---------------------------------------------------------------------------
// Fixed-order reductions.  xor-butterfly: every lane ends with the same value
// and the combination tree does not depend on timing.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum of N values per thread; result broadcast to all threads.
// scratch: >= N * 32 doubles of shared memory.
template <int N>
__device__ __forceinline__ void block_sum(double (&v)[N], double* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) scratch[i * 32 + wid] = v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = lane < nw ? scratch[i * 32 + lane] : 0.0;
    v[i] = warp_sum(s);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Grid barrier for cooperative launches (all CTAs co-resident).
// bar[0] = arrival counter, bar[1] = generation.  Release/acquire at gpu scope.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// bar[2] (when non-null callers pass bar + 2 as err) receives 1 if a CTA
// waited more than 2 s: a protocol bug must not hang the GPU.
__device__ __forceinline__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned gen = ld_acquire_gpu(bar + 1);
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == nb - 1) {
      bar[0] = 0;
      __threadfence();
      st_release_gpu(bar + 1, gen + 1);
    } else {
      const uint64_t t0 = globaltimer_ns();
      while (ld_acquire_gpu(bar + 1) == gen) {
        __nanosleep(32);
        if (globaltimer_ns() - t0 > 2000000000ull) { atomicExch(bar + 2, 1u); break; }
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Small math helpers
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Root lam >= 0 of (a^2 b s/2 + rho b^2) lam^2 + (a^2 s + 2 rho b) lam
//                 - (a S1 + b S2/2 - rho) = 0       (R17: the active-set equation
// of the elastic-net projection, derived from its KKT conditions).
__device__ __forceinline__ double enet_lambda(double a, double b, double rho, double s,
                                              double S1, double S2) {
  const double A = a * a * b * s * 0.5 + rho * b * b;
  const double B = a * a * s + 2.0 * rho * b;
  const double C = a * S1 + b * S2 * 0.5 - rho;
  const double den = B + sqrt(fmax(B * B + 4.0 * A * C, 0.0));
  return den > 0.0 ? fmax(2.0 * C / den, 0.0) : 0.0;
}

// Deterministic grid sums.  The per-atom sums S1, S2 >= 0 are accumulated as
// fixed-point integers, so the grid total does not depend on the arrival
// order of the CTAs (integer addition is associative): x in [0, 2^48)
// becomes floor(x 2^56) split in two limbs < 2^52, hi in units of 2^-4 and lo
// in units of 2^-56 (absolute resolution 1.4e-17 per CTA term, far below the
// fp32 rounding of the per-CTA partials).  Each limb sum stays < 2^60.
constexpr double kFxHi = 16.0;                       // 2^4
constexpr double kFxLo = 4503599627370496.0;         // 2^52
constexpr double kFxMax = 281474976710656.0;         // 2^48
__device__ __forceinline__ void nt_red_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// adds x into the limb pair p[0] (hi), p[1] (lo); false when x is out of range
// (negative, >= 2^48 or NaN: the sum is then clamped and the caller flags it)
__device__ __forceinline__ bool fx_red(unsigned long long* p, double x) {
  const bool ok = x >= 0.0 && x < kFxMax;
  x = ok ? x : (x >= kFxMax ? kFxMax * 0.999 : 0.0);
  const double xs = x * kFxHi;
  const double h = floor(xs);
  const unsigned long long hi = (unsigned long long)h;
  const unsigned long long lo = (unsigned long long)((xs - h) * kFxLo);
  if (hi) nt_red_u64(p, hi);
  if (lo) nt_red_u64(p + 1, lo);
  return ok;
}
__device__ __forceinline__ double fx_value(unsigned long long hi, unsigned long long lo) {
  return (double)hi * (1.0 / kFxHi) + (double)lo * (1.0 / (kFxHi * kFxLo));
}

}  // namespace somf
