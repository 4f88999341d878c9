// Microbenchmark (run by hand on a GPU box): HBM gather bandwidth of masked
// rows (~r rows apart) into shared memory with ALL of a CTA's rows in flight,
// R independent row sets per launch (launch overhead amortised), CPS CTAs
// per SM.  Modes: 0 cp.async 16 B, 2 ld.global.v4 + st.shared, 3 one
// cp.async.bulk per row (mbarrier completion, issued by one warp).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/gb2 tests/tools/gather2_bench.cu && build/gb2
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ void cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(256) gather(const float* __restrict__ src, const int* __restrict__ idx, int q,
                                              int width, int ld, int R, float* sink) {
  extern __shared__ __align__(16) float sm[];
  __shared__ __align__(8) unsigned long long mbar;
  const int G = gridDim.x, tid = threadIdx.x;
  const int lo = (int)((long long)q * blockIdx.x / G), hi = (int)((long long)q * (blockIdx.x + 1) / G);
  const int nr = hi - lo;
  float acc = 0.f;
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
  if (MODE == 3 && tid == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(mb));
  __syncthreads();
  unsigned phase = 0;
  for (int rep = 0; rep < R; ++rep) {
    const int* ix = idx + (size_t)rep * q;
    if (MODE == 0) {
      const int c4 = width / 4;
      for (int e = tid; e < nr * c4; e += blockDim.x) {
        const int r = e / c4, c = e % c4;
        cpa16(sm + r * width + 4 * c, src + (long long)ix[lo + r] * ld + 4 * c);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (MODE == 2) {
      const int c4 = width / 4;
      for (int e = tid; e < nr * c4; e += blockDim.x) {
        const int r = e / c4, c = e % c4;
        const float4 v = __ldcs(reinterpret_cast<const float4*>(src + (long long)ix[lo + r] * ld + 4 * c));
        *reinterpret_cast<float4*>(sm + r * width + 4 * c) = v;
      }
    } else {
      if (tid < 32) {
        if (tid == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"((unsigned)(nr * width * 4)) : "memory");
        __syncwarp();
        for (int r = tid; r < nr; r += 32)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"((unsigned)__cvta_generic_to_shared(sm + r * width)),
                       "l"(src + (long long)ix[lo + r] * ld), "r"((unsigned)(width * 4)), "r"(mb) : "memory");
      }
      unsigned done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(mb), "r"(phase) : "memory");
      phase ^= 1;
    }
    __syncthreads();
    acc += sm[tid % (nr * width)];
    __syncthreads();
  }
  if (acc == 1234.5f) *sink = acc;
}

int main() {
  const int p = 212445, q = 17704, R = 16;
  for (int width : {72, 200}) {
    const int ld = width;
    float* src; int* idx; float* sink;
    cudaMalloc(&src, (size_t)p * ld * 4);
    cudaMemset(src, 0, (size_t)p * ld * 4);
    std::vector<int> h((size_t)q * R);
    unsigned s = 12345;
    for (int rep = 0; rep < R; ++rep) {       // random Bernoulli-like masks: sorted random rows
      int row = 0;
      for (int i = 0; i < q; ++i) { s = s * 1664525u + 1013904223u; row += 1 + (s >> 8) % 23; h[(size_t)rep * q + i] = row % p; }
      std::vector<int> v(h.begin() + (size_t)rep * q, h.begin() + (size_t)(rep + 1) * q);
      std::sort(v.begin(), v.end());
      std::copy(v.begin(), v.end(), h.begin() + (size_t)rep * q);
    }
    cudaMalloc(&idx, (size_t)q * R * 4);
    cudaMemcpy(idx, h.data(), (size_t)q * R * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&sink, 4);
    void* flush; cudaMalloc(&flush, 256 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[] = {"cp.async16", "", "ldg.v4+sts", "bulk/row"};
    for (int cps : {1, 2, 4}) {
      const int G = 148 * cps;
      const int rows = (q + G - 1) / G;
      const size_t smem = (size_t)rows * width * 4;
      for (int mode : {0, 2, 3}) {
        void (*fn)(const float*, const int*, int, int, int, int, float*) =
            mode == 0 ? gather<0> : mode == 2 ? gather<2> : gather<3>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          cudaMemset(flush, rep, 256 << 20);
          cudaEventRecord(a);
          fn<<<G, 256, smem>>>(src, idx, q, width, ld, R, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms; cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        const double bytes = (double)q * width * 4 * R;
        printf("width %3d  CTAs/SM %d  %-12s %8.2f us  %7.1f GB/s  (%s)\n", width, cps, names[mode], best * 1e3,
               bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
    }
    cudaFree(src); cudaFree(idx); cudaFree(sink); cudaFree(flush);
  }
  return 0;
}
