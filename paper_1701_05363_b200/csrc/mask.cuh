// mask.cuh -- the random draws of one SOMF iteration (step (a0) of SURVEY §8a).
//
//  * row mask M_t (Eq. mt): row i selected iff word_{i&3} of
//    Philox((i>>2, t, 1, i>>34)) < T(r) = floor(2^32 / r)     (R1, R2)
//    -> ascending index list (P_t of P:573-577), compacted with a two-pass
//    count / scan-scatter (block-local ballot-free bit scan).
//  * atom order (Alg. 4 "permutation([1,k])"): Fisher-Yates from the
//    top with j = floor(word_w * (i+1) / 2^32), word w from Philox((w>>2, t, 2, 0)) (R13).
//  * column stream: per-epoch 6-round Feistel bijection with
//    cycle walking (R16).
#pragma once
#include "common.cuh"

namespace somf {

constexpr int kMaskThreads = 256;   // one Philox block (4 rows) per thread

// Pass 1: selected-row count per tile of kMaskThreads Philox blocks.
__global__ void __launch_bounds__(kMaskThreads)
k_mask_count(uint64_t seed, const int64_t* __restrict__ t_dev, int64_t row_lo, int64_t row_hi,
             uint64_t T, int32_t* __restrict__ tile_counts) {
  __shared__ int wsum[kMaskThreads / 32];
  const int64_t b0 = row_lo >> 2, b1 = (row_hi - 1) >> 2;
  const int64_t blk = b0 + (int64_t)blockIdx.x * kMaskThreads + threadIdx.x;
  const uint64_t t = (uint64_t)*t_dev;
  const int c = blk <= b1 ? __popc(mask_bits(seed, t, blk, row_lo, row_hi, T)) : 0;
  const int s = warp_sum(c);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < kMaskThreads / 32; ++i) tot += wsum[i];
    tile_counts[blockIdx.x] = tot;
  }
}

// Pass 2: tile base by summing the preceding tiles' counts, block-exclusive scan
// of per-thread counts, scatter of (row - idx_offset).  The last tile writes q.
__global__ void __launch_bounds__(kMaskThreads)
k_mask_scatter(uint64_t seed, const int64_t* __restrict__ t_dev, int64_t row_lo, int64_t row_hi,
               uint64_t T, const int32_t* __restrict__ tile_counts, int64_t idx_offset,
               int32_t* __restrict__ idx, int64_t* __restrict__ q_out) {
  __shared__ int64_t wpart[kMaskThreads / 32];
  __shared__ int wscan[kMaskThreads / 32];
  __shared__ int64_t base_s;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // base = sum of counts of tiles before this one (fixed order per thread, then fixed tree)
  int64_t part = 0;
  for (int i = threadIdx.x; i < (int)blockIdx.x; i += kMaskThreads) part += tile_counts[i];
  part = warp_sum(part);
  if (lane == 0) wpart[wid] = part;
  const int64_t b0 = row_lo >> 2, b1 = (row_hi - 1) >> 2;
  const int64_t blk = b0 + (int64_t)blockIdx.x * kMaskThreads + threadIdx.x;
  const uint64_t t = (uint64_t)*t_dev;
  const uint32_t bits = blk <= b1 ? mask_bits(seed, t, blk, row_lo, row_hi, T) : 0u;
  const int c = __popc(bits);
  // inclusive warp scan
  int incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wscan[wid] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t b = 0;
    for (int i = 0; i < kMaskThreads / 32; ++i) b += wpart[i];
    base_s = b;
  }
  int wbase = 0;
  for (int i = 0; i < wid; ++i) wbase += wscan[i];
  __syncthreads();
  int64_t pos = base_s + wbase + (incl - c);
  for (int l = 0; l < 4; ++l)
    if (bits & (1u << l)) idx[pos++] = (int32_t)(blk * 4 + l - idx_offset);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == kMaskThreads - 1) {
    int tot = 0;
    for (int i = 0; i < kMaskThreads / 32; ++i) tot += wscan[i];
    *q_out = base_s + tot;
  }
}

// Alg. 4's atom order by one CTA: words drawn in parallel, swaps by thread 0.
// sh: 2k words of shared memory.
__device__ __forceinline__ void atom_perm_cta(uint64_t seed, uint64_t t, int k, int cyclic,
                                              int32_t* __restrict__ perm, uint32_t* sh) {
  uint32_t* words = sh;                       // k words
  int32_t* pi = (int32_t*)(sh + k);           // k entries
  for (int i = threadIdx.x; i < k; i += blockDim.x) pi[i] = i;
  if (!cyclic) {
    for (int b = threadIdx.x; b * 4 < k - 1; b += blockDim.x) {
      const U4 w = philox4x32_10(U4{(uint32_t)b, (uint32_t)t, kStreamPerm, 0u}, seed);
      for (int l = 0; l < 4; ++l)
        if (b * 4 + l < k - 1) words[b * 4 + l] = u4_word(w, l);
    }
  }
  __syncthreads();
  if (!cyclic && threadIdx.x == 0) {
    for (int w = 0; w < k - 1; ++w) {
      const int i = k - 1 - w;
      const int j = (int)(((uint64_t)words[w] * (uint64_t)(i + 1)) >> 32);
      const int32_t tmp = pi[i];
      pi[i] = pi[j];
      pi[j] = tmp;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) perm[i] = pi[i];
}

// One launch for the start of an iteration: CTAs 0 .. ntiles-1 count the
// selected rows of M_t per tile (as k_mask_count); the extra last CTA writes
// t and the coefficients of w_t = t^-u (computed on the host) and draws the atom order (R13).
// t is passed by value (the host tracks it), so no CTA reads t_dev.
__global__ void __launch_bounds__(kMaskThreads)
k_step_mask_count(uint64_t seed, int64_t t, StepCoef cf, int64_t row_lo, int64_t row_hi, uint64_t T, int ntiles,
                  int32_t* __restrict__ tile_counts, int64_t* __restrict__ t_dev, double* __restrict__ w_dev,
                  int k, int cyclic, int32_t* __restrict__ perm) {
  __shared__ uint32_t sh[2 * 256 + 8];
  __shared__ int wsum[kMaskThreads / 32];
  if ((int)blockIdx.x == ntiles) {
    if (threadIdx.x == 0) {
      *t_dev = t;
      store_coef(w_dev, cf);          // w_t = t^-u and the mode's coefficients
    }
    atom_perm_cta(seed, (uint64_t)t, k, cyclic, perm, sh);
    return;
  }
  const int64_t b0 = row_lo >> 2, b1 = (row_hi - 1) >> 2;
  const int64_t blk = b0 + (int64_t)blockIdx.x * kMaskThreads + threadIdx.x;
  const int c = blk <= b1 ? __popc(mask_bits(seed, (uint64_t)t, blk, row_lo, row_hi, T)) : 0;
  const int s = warp_sum(c);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int i = 0; i < kMaskThreads / 32; ++i) tot += wsum[i];
    tile_counts[blockIdx.x] = tot;
  }
}

// Alg. 4's atom order, one warp: words drawn in parallel, swaps by lane 0.
__global__ void k_atom_perm(uint64_t seed, const int64_t* __restrict__ t_dev, int k, int cyclic,
                            int32_t* __restrict__ perm) {
  extern __shared__ uint32_t sh[];
  uint32_t* words = sh;                       // k words
  int32_t* pi = (int32_t*)(sh + k);           // k entries
  const uint64_t t = (uint64_t)*t_dev;
  for (int i = threadIdx.x; i < k; i += blockDim.x) pi[i] = i;
  if (!cyclic) {
    for (int b = threadIdx.x; b * 4 < k - 1; b += blockDim.x) {
      const U4 w = philox4x32_10(U4{(uint32_t)b, (uint32_t)t, kStreamPerm, 0u}, seed);
      for (int l = 0; l < 4; ++l)
        if (b * 4 + l < k - 1) words[b * 4 + l] = u4_word(w, l);
    }
  }
  __syncthreads();
  if (!cyclic && threadIdx.x == 0) {
    for (int w = 0; w < k - 1; ++w) {
      const int i = k - 1 - w;
      const int j = (int)(((uint64_t)words[w] * (uint64_t)(i + 1)) >> 32);
      const int32_t tmp = pi[i];
      pi[i] = pi[j];
      pi[j] = tmp;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) perm[i] = pi[i];
}

// Column stream: id of stream position s = pi_{s / n}(s mod n) (R16).
__global__ void k_column_ids(uint64_t seed, int64_t n, int64_t s0, int64_t count, int half,
                             int64_t* __restrict__ ids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int64_t s = s0 + i;
  const uint64_t epoch = (uint64_t)(s / n);
  const uint64_t hmask = (1ull << half) - 1;
  uint64_t x = (uint64_t)(s % n);
  do {
    uint64_t L = x >> half, R = x & hmask;
    for (int rnd = 0; rnd < 6; ++rnd) {
      const U4 w = philox4x32_10(U4{(uint32_t)R, (uint32_t)epoch, kStreamCols, (uint32_t)rnd}, seed);
      const uint64_t F = (uint64_t)w.x & hmask;
      const uint64_t nL = R;
      R = L ^ F;
      L = nL;
    }
    x = (L << half) | R;
  } while (x >= (uint64_t)n);
  ids[i] = (int64_t)x;
}

}  // namespace somf
