// Microbenchmark (run by hand on a GPU box): gather bandwidth of the masked
// rows (q rows of `width` floats, ~r rows apart) into shared memory with
// (a) 16-byte cp.async, (b) 4-byte cp.async, (c) ld.global.v4 + st.shared,
// (d) cp.async.bulk (one bulk copy per row, mbarrier completion).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/gb tests/tools/gather_bench.cu && build/gb
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void cpa16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g) : "memory");
}

// each CTA gathers rows [b*rpc, (b+1)*rpc) in chunks of 32 rows, `reps` times
template <int MODE>
__global__ void __launch_bounds__(256) gather(const float* __restrict__ src, const int* __restrict__ idx, int q,
                                              int width, int ld, float* sink) {
  extern __shared__ __align__(16) float sm[];
  __shared__ __align__(8) unsigned long long mbar;
  const int G = gridDim.x;
  const int lo = (int)((long long)q * blockIdx.x / G), hi = (int)((long long)q * (blockIdx.x + 1) / G);
  const int tid = threadIdx.x;
  float acc = 0.f;
  if (MODE == 3 && tid == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&mbar)));
  }
  __syncthreads();
  unsigned phase = 0;
  for (int r0 = lo; r0 < hi; r0 += 32) {
    const int nr = min(32, hi - r0);
    if (MODE == 0) {
      const int c4 = width / 4;
      for (int e = tid; e < nr * c4; e += 256) {
        const int r = e / c4, c = e % c4;
        cpa16(sm + r * width + 4 * c, src + (long long)idx[r0 + r] * ld + 4 * c);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (MODE == 1) {
      for (int e = tid; e < nr * width; e += 256) {
        const int r = e / width, c = e % width;
        cpa4(sm + r * width + c, src + (long long)idx[r0 + r] * ld + c);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (MODE == 2) {
      const int c4 = width / 4;
      for (int e = tid; e < nr * c4; e += 256) {
        const int r = e / c4, c = e % c4;
        const float4 v = *reinterpret_cast<const float4*>(src + (long long)idx[r0 + r] * ld + 4 * c);
        *reinterpret_cast<float4*>(sm + r * width + 4 * c) = v;
      }
    } else {
      if (tid == 0) {
        const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
        const unsigned bytes = (unsigned)(nr * width * 4);
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes) : "memory");
        for (int r = 0; r < nr; ++r) {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"((unsigned)__cvta_generic_to_shared(sm + r * width)),
                       "l"(src + (long long)idx[r0 + r] * ld), "r"((unsigned)(width * 4)), "r"(mb) : "memory");
        }
      }
      const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
      unsigned done = 0;
      while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(mb), "r"(phase) : "memory");
      }
      phase ^= 1;
    }
    __syncthreads();
    acc += sm[tid % (nr * width)];
    __syncthreads();
  }
  if (acc == 1234.5f) *sink = acc;
}

int main() {
  const int p = 212445, q = 17704;
  for (int width : {72, 200, 272}) {
    const int ld = width;
    float* src; int* idx; float* sink;
    cudaMalloc(&src, (size_t)p * ld * 4);
    cudaMemset(src, 0, (size_t)p * ld * 4);
    std::vector<int> h(q);
    for (int i = 0; i < q; ++i) h[i] = (int)((long long)i * p / q);
    cudaMalloc(&idx, q * 4);
    cudaMemcpy(idx, h.data(), q * 4, cudaMemcpyHostToDevice);
    cudaMalloc(&sink, 4);
    void* flush; cudaMalloc(&flush, 256 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const size_t smem = 32 * width * 4;
    const char* names[] = {"cp.async16", "cp.async4", "ldg.v4+sts", "bulk/row"};
    for (int mode = 0; mode < 4; ++mode) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(flush, rep, 256 << 20);
        cudaEventRecord(a);
        if (mode == 0) gather<0><<<148, 256, smem>>>(src, idx, q, width, ld, sink);
        if (mode == 1) gather<1><<<148, 256, smem>>>(src, idx, q, width, ld, sink);
        if (mode == 2) gather<2><<<148, 256, smem>>>(src, idx, q, width, ld, sink);
        if (mode == 3) gather<3><<<148, 256, smem>>>(src, idx, q, width, ld, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      const double bytes = (double)q * width * 4;
      printf("width %3d  %-12s %8.2f us  %7.1f GB/s  (%s)\n", width, names[mode], best * 1e3, bytes / best / 1e6,
             cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(src); cudaFree(idx); cudaFree(sink); cudaFree(flush);
  }
  return 0;
}
