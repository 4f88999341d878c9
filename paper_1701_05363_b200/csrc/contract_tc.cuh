// contract_tc.cuh -- (a1) the masked code step on the tensor cores:
//   beta = r D_M^T X_M (k x eta),  G = r D_M^T D_M (k x k)      (Eq. a)
// Every CTA owns ~q / #SMs masked rows and computes the partial
// [beta | G] = D_S^T [X_S | D_S] of its rows as two tcgen05 GEMMs sharing the
// A operand: M = atoms (k <= 128, padded to 128), K = masked rows (tiles of
// 128), N = eta (padded to 16; two instructions when > 256) and N = k (padded
// to 16).  3xTF32: fp32 operands are split x = hi + lo (hi exact in tf32) and
// hi.hi + hi.lo + lo.hi are accumulated in fp32 in TMEM, kind::tf32 (bf16x3
// was measured too coarse for the ridge solve at cfgC: alpha off by 2.5e-3).
// Rows arrive by 16-byte cp.async, all 128 rows of a chunk in flight at once
// ([X row | D row] raw rows, one commit group per 32 rows); each 16-row tile is
// transposed and split in shared memory into the K-major operands (a 16-byte
// K chunk = 4 rows of one atom / column) as soon as it lands, into one of two
// operand buffers: tile j + 1 is transposed while tile j's MMAs run (the
// 3xTF32 products of a 32-row tile take ~1 us of tensor time per SM, which
// was serial with the ~1 us transposition).  The partial tiles are written in fp32 and
// reduced in fixed order behind one grid barrier (ct_fused_reduce,
// cooperative launch) into r [beta | G] in fp64.
#pragma once
#include <cuda_bf16.h>
#include "common.cuh"
#include "tc_common.cuh"
#include "contract.cuh"
#include "bbar_tc.cuh"

namespace somf {

constexpr int kTcM = 128;           // atoms per accumulator (k <= 128)
constexpr int kTcK = 16;            // masked rows per tile (K of one tile)
constexpr int kTcBuf = 2;           // operand buffers: tile j + 1 is transposed / split while tile j's MMAs run
constexpr int kTcGrp = 32;          // masked rows per cp.async commit group (2 tiles)

struct CtTcArgs {
  const int32_t* idx;
  const int64_t* q_dev;
  const float* D;           // rows x kp
  int kp, k;
  const float* X;           // rows x ldx (or q x ldx when compact)
  int64_t ldx;
  int eta, xcompact;
  int ep;                   // eta rounded up to 16
  int kn;                   // k rounded up to 16 (N of the G product)
  float* partial;           // G x k x (ep + kn): [beta | pad | G | pad] rows
  CtFuse fz;
  long long* prof;          // optional: SM cycles per phase of CTA 0 (8 slots, somf_bcd_phase_cycles [224..231])
};

// fp32 -> (hi, lo) for 3xTF32: hi = x with the 13 low mantissa bits cleared
// (exactly representable in tf32), lo = x - hi (exact in fp32)
__device__ __forceinline__ void tf32_split(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

// byte offset of (row mn, k) in a K-major SWIZZLE_NONE tf32 operand of one
// tile: 16-byte chunks of 4 k, LBO = 128 (chunks adjacent), SBO = 128 kTcK / 4
__device__ __forceinline__ uint32_t tf_off(int mn, int kk) {
  return (uint32_t)((mn >> 3) * 128 * (kTcK / 4) + (kk >> 2) * 128 + (mn & 7) * 16 + (kk & 3) * 4);
}

// cp.async.wait_group with a runtime count (0..3)
__device__ __forceinline__ void cp_async_wait_upto(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
  }
}

constexpr int kTcChunk = 128;       // masked rows whose raw data is resident at once (4 tiles)

__global__ void __launch_bounds__(kCtThreads, 1) k_contract_tc(CtTcArgs P) {
  extern __shared__ __align__(128) uint8_t ctc_smem[];
  __shared__ uint32_t tmem_s;
  __shared__ __align__(8) uint64_t mbar[kTcBuf];
  __shared__ int grow[kTcChunk];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // phase clock of CTA 0, thread 0 (diagnostics; accumulated in registers, flushed once)
  const bool clk_on = P.prof && blockIdx.x == 0 && tid == 0;
  long long t_mark = clock64(), t_ph[7] = {0, 0, 0, 0, 0, 0, 0};
#define CTC_MARK(slot)                 \
  do {                                 \
    if (clk_on) {                      \
      const long long now_ = clock64(); \
      t_ph[slot] += now_ - t_mark;     \
      t_mark = now_;                   \
    }                                  \
  } while (0)
  const int k = P.k, kp = P.kp, eta = P.eta, ep = P.ep, kn = P.kn;
  const int LDR = ep + kp;                            // raw row: [X row (ep) | D row (kp)]
  const int G = gridDim.x;
  const int64_t q = *P.q_dev;
  const int64_t lo = q * blockIdx.x / G, hi = q * (blockIdx.x + 1) / G;
  const size_t a_bytes = (size_t)kTcM * kTcK * 4, x_bytes = (size_t)ep * kTcK * 4;
  const size_t set_bytes = 2 * (a_bytes + x_bytes);   // one operand buffer: A hi / lo, X hi / lo
  // buffer b: Ahi (atoms x rows, K-major tf32) | Alo | Xhi (X columns x rows) | Xlo
  float* raw = reinterpret_cast<float*>(ctc_smem + kTcBuf * set_bytes);   // kTcChunk x LDR (fp32 rows)
  // TMEM: columns [0, ep) beta, [ep, ep + kn) G
  const uint32_t ncols = (ep + kn) <= 256 ? 256 : 512;
  if (wid == 0) tc_alloc(&tmem_s, ncols);
  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < kTcBuf; ++b) mbar_init(&mbar[b], 1);
  }
  // Warp roles in the tile loop: warps 0..6 (kTcWorkers threads) gather,
  // transpose and split; warp 7 only issues the MMAs (a tile's 12 tcgen05.mma
  // take ~0.5 us to issue -- as long as its transposition -- so an issuing
  // thread that also transposes would serialise the two).  Named barriers:
  // 1 = workers only; 2 + b = "operands of buffer b stored" (workers arrive
  // without waiting, the MMA warp syncs).
  constexpr int kTcWorkers = kCtThreads - 32;
  const bool worker = tid < kTcWorkers;
  auto bar_workers = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(kTcWorkers) : "memory"); };
  uint32_t phase_bits = 0;                            // bit b: parity of buffer b's mbarrier
  uint32_t pend_bits = 0;                             // bit b: MMAs committed on buffer b, not yet waited for
  int jt = 0;                                         // tiles issued so far (buffer = jt % kTcBuf)
  const uint64_t dbase = tc_sdesc(ctc_smem, 128, 128u * (kTcK / 4));
  const uint32_t idg = tc_idesc_tf32(kTcM, kn);
  const int cx = eta / 4, cd = kp / 4, cr = cx + cd;  // 16-byte chunks of a raw row (eta % 4 == 0)
  tc_sync_before();
  __syncthreads();                                    // TMEM address, mbarriers initialised
  tc_sync_after();
  long long t_issue = 0;                              // MMA warp, lane 0: cycles spent issuing
  for (int64_t c0 = lo; c0 < hi; c0 += kTcChunk) {
    const int nrow = (int)(hi - c0 < (int64_t)kTcChunk ? hi - c0 : (int64_t)kTcChunk);
    const int ntile = (nrow + kTcK - 1) / kTcK, ngrp = (nrow + kTcGrp - 1) / kTcGrp;
    if (!worker) {
      // ---- MMA warp: per tile, wait for its operands, issue, commit ----
      for (int j = 0; j < ntile; ++j, ++jt) {
        const int b = jt % kTcBuf;
        asm volatile("bar.sync %0, %1;" ::"r"(2 + b), "r"(kCtThreads) : "memory");
        tc_sync_after();
        if (lane == 0) {
          const long long ti0 = P.prof && blockIdx.x == 0 ? clock64() : 0;
          const uint32_t tmem = tmem_s;
          // descriptors: buffer 0's Ahi descriptor + 16-byte offsets (the address
          // field holds addr >> 4; no carry out of it below 256 KB of shared memory)
          const uint64_t dAh = dbase + (uint64_t)(((size_t)b * set_bytes) >> 4), dAl = dAh + (a_bytes >> 4);
          const uint64_t dXh = dAl + (a_bytes >> 4), dXl = dXh + (x_bytes >> 4);
          const bool first = jt == 0;
#pragma unroll
          for (int ks = 0; ks < kTcK / 8; ++ks) {
            const uint64_t kq = (uint64_t)ks * 16;    // 256 bytes of K per instruction
            const uint64_t ah = dAh + kq, al = dAl + kq;
            const bool acc0 = !first || ks > 0;
            // beta: N = ep in pieces of <= 256 (multiples of 16)
            for (int n0 = 0; n0 < ep; n0 += 256) {
              const int nn = ep - n0 < 256 ? ep - n0 : 256;
              const uint32_t id = tc_idesc_tf32(kTcM, nn);
              const uint64_t xo = kq + (uint64_t)n0 * (kTcK / 4);        // n0 rows of 16 (kTcK / 4) bytes
              tc_mma_tf32(tmem + n0, ah, dXh + xo, id, acc0);
              tc_mma_tf32(tmem + n0, ah, dXl + xo, id, true);
              tc_mma_tf32(tmem + n0, al, dXh + xo, id, true);
            }
            // G: B = the same D rows (the A operand), N = kn
            tc_mma_tf32(tmem + ep, ah, ah, idg, acc0);
            tc_mma_tf32(tmem + ep, ah, al, idg, true);
            tc_mma_tf32(tmem + ep, al, ah, idg, true);
          }
          tc_commit(&mbar[b]);
          if (P.prof && blockIdx.x == 0) t_issue += clock64() - ti0;
        }
        __syncwarp();
      }
      continue;
    }
    // ---- workers ----
    // (the previous chunk's raw rows were last read by the transposition of
    // its last tile, before that tile's arrive; this barrier orders them)
    bar_workers();
    for (int r = tid; r < kTcChunk; r += kTcWorkers) grow[r] = r < nrow ? P.idx[c0 + r] : -1;
    bar_workers();
    // every row of the chunk in flight at once: one commit group per 32 rows
    for (int g = 0; g < ngrp; ++g) {
      const int r0 = g * kTcGrp, r1 = min(nrow, r0 + kTcGrp);
      for (int e = tid; e < (r1 - r0) * cr; e += kTcWorkers) {
        const int r = r0 + e / cr, c = e % cr;
        const int64_t gr = grow[r];
        const float* src =
            c < cx ? P.X + (P.xcompact ? c0 + r : gr) * P.ldx + 4 * c : P.D + gr * kp + 4 * (c - cx);
        float* dst = raw + (size_t)r * LDR + (c < cx ? 4 * c : ep + 4 * (c - cx));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    CTC_MARK(0);                                      // row indices + cp.async issue
    for (int j = 0; j < ntile; ++j, ++jt) {
      const int b = jt % kTcBuf;
      uint8_t* Ahi = ctc_smem + (size_t)b * set_bytes;
      uint8_t* Alo = Ahi + a_bytes;
      uint8_t* Xhi = Alo + a_bytes;
      uint8_t* Xlo = Xhi + x_bytes;
      if ((j * kTcK) % kTcGrp == 0) {
        cp_async_wait_upto(ngrp - 1 - (j * kTcK) / kTcGrp);
        CTC_MARK(1);                                  // rows of the group landed (mine)
        bar_workers();                                // ... and every worker's
      }
      if ((pend_bits >> b) & 1u) {                    // tile jt - 2's MMAs have read this operand buffer
        mbar_wait(&mbar[b], (phase_bits >> b) & 1u);
        phase_bits ^= 1u << b;
        pend_bits &= ~(1u << b);
      }
      CTC_MARK(2);                                    // group barrier + this buffer's previous MMAs
      // ---- transpose + split tile j into K-major tf32 hi / lo operands ----
      // thread -> one operand row m (atom, or X column), all kTcK / 4 chunks
      for (int m = tid; m < kTcM + ep; m += kTcWorkers) {
        const bool isA = m < kTcM;
        const int col = isA ? ep + m : m - kTcM;     // column of the raw row
        const bool valid = isA ? m < k : col < eta;
        float v[kTcK];
#pragma unroll
        for (int r = 0; r < kTcK; ++r) {
          const int rr = j * kTcK + r;
          v[r] = (valid && rr < nrow) ? raw[(size_t)rr * LDR + col] : 0.f;
        }
        uint8_t* hb = isA ? Ahi : Xhi;
        uint8_t* lb = isA ? Alo : Xlo;
        const int mm = isA ? m : m - kTcM;
#pragma unroll
        for (int c = 0; c < kTcK / 4; ++c) {
          float4 h, l;
          tf32_split(v[4 * c + 0], h.x, l.x);
          tf32_split(v[4 * c + 1], h.y, l.y);
          tf32_split(v[4 * c + 2], h.z, l.z);
          tf32_split(v[4 * c + 3], h.w, l.w);
          const uint32_t off = tf_off(mm, 4 * c);
          *reinterpret_cast<float4*>(hb + off) = h;
          *reinterpret_cast<float4*>(lb + off) = l;
        }
      }
      CTC_MARK(3);                                    // transpose + split
      tc_fence_smem_to_async();
      asm volatile("bar.arrive %0, %1;" ::"r"(2 + b), "r"(kCtThreads) : "memory");
      pend_bits |= 1u << b;
    }
  }
  // MMAs complete in issue order, commits arrive in order: the workers wait for
  // both buffers; the CTA barrier then covers the MMA warp
  if (worker) {
#pragma unroll
    for (int b = 0; b < kTcBuf; ++b)
      if ((pend_bits >> b) & 1u) mbar_wait(&mbar[b], (phase_bits >> b) & 1u);
  }
  tc_sync_before();
  __syncthreads();
  tc_sync_after();
  CTC_MARK(2);
  const int ntile_all = hi > lo ? 1 : 0;
  // ---- epilogue: partial tile [beta | pad | G | pad] of my rows (fp32), lane = atom ----
  const int ncp = ep + kn;
  float* out = P.partial + (int64_t)blockIdx.x * k * ncp;
  if (ntile_all > 0) {
    // TMEM -> shared memory (lane = atom row, 16 columns per tcgen05.ld; row
    // stride ncp + 4 words so the 16-byte stores of a quarter-warp cover all
    // banks) -> global memory with consecutive threads on consecutive 16 bytes
    // (a direct store from the TMEM fragment is 32 scattered 16-byte requests
    // per instruction: 4.6 us for the 80 KB tile at cfgC).  The operand
    // buffers and raw rows are free: every MMA has completed.
    float* stage = reinterpret_cast<float*>(ctc_smem);
    const int lds = ncp + 4;
    const int a = 32 * (wid & 3) + lane;
    const uint32_t tl = tmem_s + ((uint32_t)(32 * (wid & 3)) << 16);
    const int nchunk = ncp / 16;
    for (int cc = wid >> 2; cc < nchunk; cc += 2) {
      float v[16];
      tc_ld16(tl + 16 * cc, v);
      if (a < k) {
        float4* o4 = reinterpret_cast<float4*>(stage + (size_t)a * lds + 16 * cc);
#pragma unroll
        for (int j = 0; j < 4; ++j) o4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      }
    }
    __syncthreads();
    const int n4 = ncp / 4;
    for (int e = tid; e < k * n4; e += kCtThreads) {
      const int r = e / n4, c = e % n4;
      reinterpret_cast<float4*>(out)[e] = *reinterpret_cast<const float4*>(stage + (size_t)r * lds + 4 * c);
    }
  } else {
    for (int e = tid; e < k * ncp; e += kCtThreads) out[e] = 0.f;
  }
  tc_sync_before();
  __syncthreads();
  if (wid == 0) tc_dealloc(tmem_s, ncols);
  CTC_MARK(4);                                        // epilogue: TMEM -> fp32 partial tile
  long long t_bar = 0;
  ct_fused_reduce(P.partial, k, eta, ep + kn, ep, P.fz, reinterpret_cast<double*>(ctc_smem),
                  clk_on ? &t_bar : nullptr);
  if (clk_on) {
    CTC_MARK(6);                                      // barrier + fixed-order reduction
    t_ph[5] = t_bar;                                  // the grid barrier's share
    t_ph[6] -= t_bar;
#pragma unroll
    for (int i = 0; i < 7; ++i) P.prof[i] += t_ph[i];
    P.prof[7] += 1;
  }
  if (P.prof && blockIdx.x == 0 && tid == kTcWorkers) P.prof[17] += t_issue;    // slot 241: MMA issue (MMA warp)
#undef CTC_MARK
}

}  // namespace somf
