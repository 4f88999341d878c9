// umma_probe.cu -- checks the hand-built tcgen05 (UMMA) descriptors used by
// csrc/tc_common.cuh on the GPU: D[M x N] = A[M x K] B[N x K]^T with both
// operands K-major, SWIZZLE_NONE (INTERLEAVE) layout, fp32 accumulator in
// TMEM, for kind::f16 (bf16 inputs, K = 16 per instruction) and kind::tf32
// (K = 8 per instruction).  Prints the max relative error vs a CPU reference.
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a tests/tools/umma_probe.cu -o /tmp/umma_probe
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>

#include "../../paper_1701_05363_b200/csrc/tc_common.cuh"

using namespace somf;

constexpr int M = 128, N = 64, K = 64;

// MN-major tf32 candidates (T = 4 elements per 16 bytes):
//  var 0: [MN grp][K grp][k%8][16B]  lbo = 128 (K grp), sbo = 128*K/8 (MN grp)
//  var 1: same data, fields swapped  lbo = 128*K/8, sbo = 128
//  var 2: [K grp][MN grp][k%8][16B]  lbo = 128*MN/4 (K grp), sbo = 128 (MN grp)
//  var 3: same data as 2, swapped    lbo = 128, sbo = 128*MN/4
__device__ size_t mn_off(int mn, int k, int var) {
  if (var < 2) return (size_t)(mn / 4) * 128 * (K / 8) + (size_t)(k / 8) * 128 + (k % 8) * 16 + (mn % 4) * 4;
  return (size_t)(k / 8) * 128 * (128 / 4) + (size_t)(mn / 4) * 128 + (k % 8) * 16 + (mn % 4) * 4;
}
__device__ uint64_t mn_desc(uint8_t* base, int ks, int var, int nmn) {
  (void)nmn;
  switch (var) {
    case 0: return tc_sdesc(base + (size_t)ks * 128, 128, 128 * (K / 8));
    case 1: return tc_sdesc(base + (size_t)ks * 128, 128 * (K / 8), 128);
    case 2: return tc_sdesc(base + (size_t)ks * 128 * 32, 128 * 32, 128);
    default: return tc_sdesc(base + (size_t)ks * 128 * 32, 128, 128 * 32);
  }
}

template <bool kTf32, bool kMN>
__global__ void probe(const float* A, const float* B, float* D, int var) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  constexpr int ES = kTf32 ? 4 : 2;               // element bytes
  constexpr int T = 16 / ES;                      // elements per 16-byte chunk
  constexpr int NCH = K / T;                      // K chunks
  uint8_t* As = smem;
  uint8_t* Bs = smem + (size_t)M * K * ES;   // (var 2/3 lay B out with 128 MN rows)
  const int tid = threadIdx.x;
  // K-major: [group g][chunk c][row r][16B]: LBO = 128 (chunk), SBO = 128 * NCH (8-row group)
  // MN-major (tf32): [MN group of T][K group of 8][k % 8][16B]: LBO = 128, SBO = 128 * K / 8
  for (int e = tid; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    const size_t off = kMN ? mn_off(m, k, var) : (size_t)(m / 8) * 128 * NCH + (size_t)(k / T) * 128 + (m % 8) * 16 + (k % T) * ES;
    if (kTf32) *reinterpret_cast<float*>(As + off) = A[e];
    else *reinterpret_cast<__nv_bfloat16*>(As + off) = __float2bfloat16(A[e]);
  }
  for (int e = tid; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e % K;
    const size_t off = kMN ? mn_off(n, k, var) : (size_t)(n / 8) * 128 * NCH + (size_t)(k / T) * 128 + (n % 8) * 16 + (k % T) * ES;
    if (kTf32) *reinterpret_cast<float*>(Bs + off) = B[e];
    else *reinterpret_cast<__nv_bfloat16*>(Bs + off) = __float2bfloat16(B[e]);
  }
  if (tid < 32) tc_alloc(&tmem_base, 64);
  if (tid == 0) mbar_init(&mbar, 1);
  tc_fence_smem_to_async();
  tc_sync_before();
  __syncthreads();
  tc_sync_after();
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t idesc = (kTf32 ? tc_idesc_tf32(M, N) : tc_idesc_bf16(M, N)) | (kMN ? (3u << 15) : 0u);
    constexpr int KSTEP = kTf32 ? 8 : 16;         // K per instruction = 2 chunks (K-major) / 1 K group (MN)
    for (int ks = 0; ks < K / KSTEP; ++ks) {
      const uint64_t ad = kMN ? mn_desc(As, ks, var, M) : tc_sdesc(As + (size_t)ks * 2 * 128, 128, 128 * NCH);
      const uint64_t bd = kMN ? mn_desc(Bs, ks, var, N) : tc_sdesc(Bs + (size_t)ks * 2 * 128, 128, 128 * NCH);
      if (kTf32) tc_mma_tf32(tmem, ad, bd, idesc, ks > 0);
      else tc_mma_bf16(tmem, ad, bd, idesc, ks > 0);
    }
    tc_commit(&mbar);
  }
  mbar_wait(&mbar, 0);
  tc_sync_after();
  // warp w reads lanes 32w..32w+31 (rows), N columns
  const int w = tid >> 5, lane = tid & 31;
  if (w < 4) {
    for (int c0 = 0; c0 < N; c0 += 16) {
      float v[16];
      tc_ld16(tmem + ((uint32_t)(32 * w) << 16) + c0, v);
      for (int j = 0; j < 16; ++j) D[(size_t)(32 * w + lane) * N + c0 + j] = v[j];
    }
  }
  tc_sync_before();
  __syncthreads();
  if (tid < 32) tc_dealloc(tmem, 64);
}

static float bf(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x7fff + ((u >> 16) & 1);
  u &= 0xffff0000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

template <bool kTf32, bool kMN = false>
static int run(int var = 0) {
  std::vector<float> A(M * K), B(N * K), D(M * N);
  srand(1);
  for (auto& x : A) x = (float)rand() / RAND_MAX - 0.5f;
  for (auto& x : B) x = (float)rand() / RAND_MAX - 0.5f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = (size_t)(M + 128) * K * (kTf32 ? 4 : 2);
  cudaFuncSetAttribute(probe<kTf32, kMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<kTf32, kMN><<<1, 128, smem>>>(dA, dB, dD, var);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("%s: CUDA error %s\n", kTf32 ? "tf32" : "bf16", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) {
        const float a = kTf32 ? A[m * K + k] : bf(A[m * K + k]), b = kTf32 ? B[n * K + k] : bf(B[n * K + k]);
        r += (double)a * b;
      }
      maxerr = fmax(maxerr, fabs(r - D[m * N + n]));
      maxref = fmax(maxref, fabs(r));
    }
  printf("%s%s var %d: max |err| %.3e (max |ref| %.3e) -> %s\n", kTf32 ? "tf32" : "bf16", kMN ? " MN-major" : "", var, maxerr, maxref,
         maxerr <= (kTf32 ? 2e-2 : 1e-3) * maxref ? "OK" : "MISMATCH");
  return maxerr <= (kTf32 ? 2e-2 : 1e-3) * maxref ? 0 : 1;
}

int main() {
  int bad = run<false>();
  bad |= run<true>();
  for (int v = 0; v < 4; ++v) run<true, true>(v);
  return bad;
}
