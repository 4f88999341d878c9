// bbar_tc.cuh -- (a3) masked-row surrogate aggregation on the tensor cores:
//   P_t Bbar <- (1 - w) P_t Bbar + (w / eta) X_M A^T      (Eq. somf_partial
//   P:602, masked rows only (north star), batch mean R4)
// as one tcgen05 GEMM per tile of 128 masked rows: D[rows x k] = X_M[rows x eta]
// . A[k x eta]^T, fp32 accumulator in TMEM.  fp32 operands are split into two
// bf16 terms (x = hi + lo, |x - hi - lo| <= 2^-17 |x|) and three products
// hi.hi + hi.lo + lo.hi are accumulated (bf16x3: per-product error ~2^-16,
// DESIGN.md §5), kind::f16, K = 16 per instruction.
//
// One CTA per SM owns ~q / #SMs masked rows (tiles of 128).  Staging: the
// codes (B operand, N = k rounded up to 16) once per CTA, the masked X rows
// (A operand, M = 128) per tile, both written split and in the K-major
// SWIZZLE_NONE core-matrix layout of tc_common.cuh; the old Bbar rows by
// cp.async.  Thread 0 issues the 3 x ceil(eta/16) MMAs, commits to an
// mbarrier; the epilogue (warp w: TMEM lanes 32 (w % 4) .., column half w / 4)
// reads the accumulator and writes keep * Bbar_old + add * acc.
// Optionally folds the Cbar update (CbarFold, as k_bbar_v3).
#pragma once
#include <cuda_bf16.h>
#include "common.cuh"
#include "tc_common.cuh"
#include "bbar.cuh"

namespace somf {

constexpr int kBtThreads = 256;
constexpr int kBtM = 128;

struct BtArgs {
  const int32_t* idx;       // masked local rows (ascending): the Bbar rows; null = every row (mode F)
  int xcompact;             // X holds only the masked rows (row m of X = m-th masked row)
  const int64_t* q_dev;
  const float* X;           // rows x ldx (or q x ldx when compact)
  int64_t ldx;
  int eta, k, kp;
  const float* A;           // codes k x eta (fp32, row-major)
  float* Bbar;              // rows x kp
  const double* w_dev;
  int np;                   // N: k rounded up to 16
  int ep;                   // eta rounded up to 16
  CbarFold cf;
  int pdl;                  // launched as a programmatic dependent of the code solver
  long long* prof;          // optional: SM cycles per phase of CTA 0 (8 slots, somf_bcd_phase_cycles [232..239])
};

__device__ __forceinline__ void bt_split(float x, __nv_bfloat16& hi, __nv_bfloat16& lo) {
  hi = __float2bfloat16_rn(x);
  lo = __float2bfloat16_rn(x - __bfloat162float(hi));
}

// one 16-byte K chunk (8 values) of one operand row: split and store hi / lo
__device__ __forceinline__ void bt_store_chunk(const float (&v)[8], uint8_t* hi_base, uint8_t* lo_base,
                                               uint32_t off) {
  __align__(16) __nv_bfloat16 h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) bt_split(v[i], h[i], l[i]);
  *reinterpret_cast<uint4*>(hi_base + off) = *reinterpret_cast<const uint4*>(h);
  *reinterpret_cast<uint4*>(lo_base + off) = *reinterpret_cast<const uint4*>(l);
}

// 8 consecutive floats of a row of length len starting at s (zeros past len)
__device__ __forceinline__ void bt_load8(const float* row, int s, int len, bool streaming, float (&v)[8]) {
  if (s + 8 <= len && ((reinterpret_cast<uintptr_t>(row + s) & 15) == 0)) {
    const float4 a = streaming ? __ldcs(reinterpret_cast<const float4*>(row + s))
                               : __ldg(reinterpret_cast<const float4*>(row + s));
    const float4 b = streaming ? __ldcs(reinterpret_cast<const float4*>(row + s + 4))
                               : __ldg(reinterpret_cast<const float4*>(row + s + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = s + i < len ? row[s + i] : 0.f;
  }
}

// byte offset of element (row, kk) in a K-major SWIZZLE_NONE bf16 operand with
// LBO = 128 (K chunks adjacent) and SBO = 128 * nch (8-row groups)
__device__ __forceinline__ uint32_t bt_off(int row, int kk, int nch) {
  return (uint32_t)((row >> 3) * 128 * nch + (kk >> 3) * 128 + (row & 7) * 16 + (kk & 7) * 2);
}

__global__ void __launch_bounds__(kBtThreads, 1) k_bbar_tc(BtArgs P) {
  // the BCD kernel may launch now (programmatic dependent launch): its CTAs
  // take an SM as soon as my CTA there exits, and read what I write only
  // after griddepcontrol.wait
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ __align__(128) uint8_t bt_smem[];
  __shared__ uint32_t tmem_s;
  __shared__ __align__(8) uint64_t mbar;
  __shared__ int grow[kBtM];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // phase clock of CTA 0, thread 0 (diagnostics; accumulated in registers, flushed once)
  const bool clk_on = P.prof && blockIdx.x == 0 && tid == 0;
  long long t_mark = clock64(), t_ph[7] = {0, 0, 0, 0, 0, 0, 0};
#define BT_MARK(slot)                   \
  do {                                  \
    if (clk_on) {                       \
      const long long now_ = clock64(); \
      t_ph[slot] += now_ - t_mark;      \
      t_mark = now_;                    \
    }                                   \
  } while (0)
  const int eta = P.eta, k = P.k, kp = P.kp, np = P.np, ep = P.ep, nch = ep / 8;
  const int G = gridDim.x;
  const int64_t q = *P.q_dev;
  const double keepd = P.w_dev[kCoefKeep], gb = P.w_dev[kCoefGainB], gc = P.w_dev[kCoefGainC];
  const float keep = (float)keepd, add = (float)(gb / eta);
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  const size_t a_bytes = (size_t)kBtM * ep * 2, b_bytes = (size_t)np * ep * 2;
  uint8_t* Ahi = bt_smem;
  uint8_t* Alo = Ahi + a_bytes;
  uint8_t* Bhi = Alo + a_bytes;
  uint8_t* Blo = Bhi + b_bytes;
  float* Bold = reinterpret_cast<float*>(Blo + b_bytes);        // 128 x kp
  // Everything the code solver writes (the codes A, the Cbar partials) is read
  // only after griddepcontrol.wait: with programmatic dependent launch the CTAs
  // start while the solver still runs and stage their first tile of X rows and
  // old Bbar rows (written by earlier kernels) in the meantime.  The Cbar
  // update runs AFTER the first tile's MMAs are issued (under the tensor pipe
  // and the old-Bbar cp.async), off the path wait -> codes -> MMA -> epilogue.
  auto wait_solver = [&]() {
    if (P.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  };
  auto fold_cbar = [&]() {
    if (P.cf.A64) {
      // my slice of the Cbar entries (Eq. somf_partial) straight from the
      // fp64 codes: sum_s a_s a_s^T, s in column order, 8 threads per entry
      // (strided columns) combined in fixed order.  Only the lower triangle
      // (a >= b) is summed; entry (b, a) gets the same bits (the products
      // commute), so Cbar stays exactly symmetric and a CTA's slice
      // (k (k + 1) / 2 / G entries: 17 at cfgC) is one pass of 32 entries.
      const int kq = P.cf.k, ne = P.cf.eta;
      const int ntri = kq * (kq + 1) / 2;
      const int e0 = (int)((int64_t)ntri * blockIdx.x / G), e1 = (int)((int64_t)ntri * (blockIdx.x + 1) / G);
      for (int eb = e0; eb < e1; eb += kBtThreads / 8) {
        const int e = eb + tid / 8, h = tid % 8;
        double s = 0.0;
        int ia = 0, ib = 0;
        if (e < e1) {
          // e = ia (ia + 1) / 2 + ib, ib <= ia
          ia = (int)((sqrtf(8.f * (float)e + 1.f) - 1.f) * 0.5f);
          while (ia * (ia + 1) / 2 > e) --ia;
          while ((ia + 1) * (ia + 2) / 2 <= e) ++ia;
          ib = e - ia * (ia + 1) / 2;
          const double* ra = P.cf.A64 + (int64_t)ia * ne;
          const double* rb = P.cf.A64 + (int64_t)ib * ne;
#pragma unroll 8
          for (int c = h; c < ne; c += 8) s = fma(__ldg(ra + c), __ldg(rb + c), s);
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        if (e < e1 && h == 0) {
          const int eab = ia * kq + ib, eba = ib * kq + ia;
          const double c = keepd * P.cf.C64[eab] + (gc / eta) * s;
          P.cf.C64[eab] = c;
          P.cf.C32[eab] = (float)c;
          if (ia != ib) {
            P.cf.C64[eba] = c;
            P.cf.C32[eba] = (float)c;
          }
        }
      }
    } else if (P.cf.cpart) {
      // my slice of the Cbar entries (Eq. somf_partial)
      const int e0 = (int)((int64_t)P.cf.kk * blockIdx.x / G), e1 = (int)((int64_t)P.cf.kk * (blockIdx.x + 1) / G);
      for (int e = e0 + tid; e < e1; e += kBtThreads) {
        double s = 0.0;
        for (int bq = 0; bq < P.cf.nparts; ++bq) s += P.cf.cpart[(size_t)bq * P.cf.kk + e];
        const double c = keepd * P.cf.C64[e] + (gc / eta) * s;
        P.cf.C64[e] = c;
        P.cf.C32[e] = (float)c;
      }
    }
  };
  if (hi <= lo) {
    wait_solver();
    fold_cbar();
    return;
  }
  if (wid == 0) tc_alloc(&tmem_s, np <= 32 ? 32 : np <= 64 ? 64 : np <= 128 ? 128 : 256);
  if (tid == 0) mbar_init(&mbar, 1);
  bool waited = false, folded = false;
  const uint32_t idesc = tc_idesc_bf16(kBtM, np);
  uint32_t phase = 0;
  for (int64_t t0 = lo; t0 < hi; t0 += kBtM) {
    const int n = (int)(hi - t0 < (int64_t)kBtM ? hi - t0 : (int64_t)kBtM);
    __syncthreads();                                   // previous tile's epilogue done with smem
    for (int r = tid; r < kBtM; r += kBtThreads) grow[r] = r < n ? (P.idx ? P.idx[t0 + r] : (int)(t0 + r)) : 0;
    __syncthreads();
    // old Bbar rows of the tile (async; consumed by the epilogue)
    for (int e = tid; e < n * (kp / 4); e += kBtThreads) {
      const int r = e / (kp / 4), c = e % (kp / 4);
      const unsigned d = smem_u32(Bold + (size_t)r * kp + 4 * c);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                   "l"(P.Bbar + (int64_t)grow[r] * kp + 4 * c)
                   : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // A = masked X rows (M = 128 x K = ep), split.  A warp's 32 items are 8
    // rows x 4 consecutive K chunks: the loads read 128 contiguous bytes of
    // each row (8 lines per instruction instead of 32 scattered sectors) and
    // the 16-byte stores cover 512 contiguous bytes (conflict-free); U chunks
    // of every thread in flight before the stores (the gather is
    // latency-bound: one round of loads, not several)
    {
      constexpr int U = 14;                         // every chunk of a thread in flight (eta <= 224)
      const int ncg = (nch + 3) / 4;                // groups of 4 chunks
      auto item = [&](int e, int& r, int& c) {
        const int blk = e >> 5;
        r = (blk % (kBtM / 8)) * 8 + (e & 7);
        c = (blk / (kBtM / 8)) * 4 + ((e >> 3) & 3);
      };
      for (int e0 = tid; e0 < kBtM * 4 * ncg; e0 += kBtThreads * U) {
        float v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kBtThreads;
          int r, c;
          item(e, r, c);
          if (e < kBtM * 4 * ncg && c < nch && r < n) {
            const int64_t xr = P.xcompact ? t0 + r : (int64_t)grow[r];
            bt_load8(P.X + xr * P.ldx, 8 * c, eta, true, v[u]);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[u][i] = 0.f;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kBtThreads;
          int r, c;
          item(e, r, c);
          if (e < kBtM * 4 * ncg && c < nch) bt_store_chunk(v[u], Ahi, Alo, bt_off(r, 8 * c, nch));
        }
      }
    }
    BT_MARK(0);                                        // X rows gathered, split, stored (+ old Bbar issue)
    if (!waited) {
      wait_solver();
      BT_MARK(1);                                      // waiting for the code solver
      waited = true;
      // ---- B = codes (N = np x K = ep), split, once per CTA ----
      // (UB chunks of a thread in flight before the stores: the codes sit in
      // L2 and the loop is latency-bound -- one round trip, not np nch / 256)
      {
        constexpr int UB = 9;
        for (int e0 = tid; e0 < np * nch; e0 += kBtThreads * UB) {
          float v[UB][8];
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int e = e0 + u * kBtThreads;
            const int n = e % np, c = e / np;          // n fastest: conflict-free 16-byte stores
            if (e < np * nch && n < k) bt_load8(P.A + (int64_t)n * eta, 8 * c, eta, false, v[u]);
            else
#pragma unroll
              for (int i = 0; i < 8; ++i) v[u][i] = 0.f;
          }
#pragma unroll
          for (int u = 0; u < UB; ++u) {
            const int e = e0 + u * kBtThreads;
            if (e < np * nch) bt_store_chunk(v[u], Bhi, Blo, bt_off(e % np, 8 * (e / np), nch));
          }
        }
      }
    }
    tc_fence_smem_to_async();
    tc_sync_before();
    __syncthreads();
    tc_sync_after();
    BT_MARK(2);                                        // codes staged (B operand)
    const uint32_t tmem = tmem_s;
    if (tid == 0) {
      // D = Ahi Bhi^T + Ahi Blo^T + Alo Bhi^T over K = ep (2 chunks of 8 per instruction)
      const uint32_t sbo_a = 128u * nch, sbo_b = 128u * nch;
      for (int ks = 0; ks < ep / 16; ++ks) {
        const size_t ko = (size_t)ks * 256;
        const uint64_t ah = tc_sdesc(Ahi + ko, 128, sbo_a), al = tc_sdesc(Alo + ko, 128, sbo_a);
        const uint64_t bh = tc_sdesc(Bhi + ko, 128, sbo_b), bl = tc_sdesc(Blo + ko, 128, sbo_b);
        tc_mma_bf16(tmem, ah, bh, idesc, ks > 0);
        tc_mma_bf16(tmem, ah, bl, idesc, true);
        tc_mma_bf16(tmem, al, bh, idesc, true);
      }
      tc_commit(&mbar);
    }
    BT_MARK(3);                                        // MMA issue
    if (!folded) {
      fold_cbar();
      folded = true;
    }
    BT_MARK(4);                                        // Cbar update
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    mbar_wait(&mbar, phase);
    phase ^= 1;
    __syncthreads();                                   // Bold rows of every thread landed
    tc_sync_after();
    BT_MARK(5);                                        // MMAs done, old rows landed
    // ---- epilogue: warp w reads lanes 32 (w % 4) .. (rows), column half w / 4 ----
    {
      const int row = 32 * (wid & 3) + lane;
      const int nck = np / 16, c0 = (wid >> 2) * ((nck + 1) / 2), c1 = min(nck, c0 + (nck + 1) / 2);
      for (int cc = c0; cc < c1; ++cc) {
        float v[16];
        tc_ld16(tmem + ((uint32_t)(32 * (wid & 3)) << 16) + 16 * cc, v);
        if (row < n) {
          // 16-byte stores up to kp (padding columns stay 0: zero codes, zero old values)
          float* brow = P.Bbar + (int64_t)grow[row] * kp;
          const float* bo = Bold + (size_t)row * kp;
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            const int a0 = 16 * cc + 4 * j4;
            if (a0 + 4 <= kp) {
              const float4 o = *reinterpret_cast<const float4*>(bo + a0);
              *reinterpret_cast<float4*>(brow + a0) =
                  make_float4(fmaf(keep, o.x, add * v[4 * j4]), fmaf(keep, o.y, add * v[4 * j4 + 1]),
                              fmaf(keep, o.z, add * v[4 * j4 + 2]), fmaf(keep, o.w, add * v[4 * j4 + 3]));
            }
          }
        }
      }
    }
    tc_sync_before();
    BT_MARK(6);                                        // epilogue: TMEM -> keep * old + add * acc -> Bbar rows
  }
  __syncthreads();
  if (wid == 0) tc_dealloc(tmem_s, np <= 32 ? 32 : np <= 64 ? 64 : np <= 128 ? 128 : 256);
  if (clk_on) {
#pragma unroll
    for (int i = 0; i < 7; ++i) P.prof[i] += t_ph[i];
    P.prof[7] += 1;
  }
#undef BT_MARK
}

}  // namespace somf
