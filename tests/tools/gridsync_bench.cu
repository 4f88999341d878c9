// Microbenchmark: cost of one grid-wide reduction round on B200, the unit
// of latency of the on-chip BCD kernel (bcd_onchip.cuh).  Not part of the
// library; built and run by hand on a GPU box:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/gs tests/tools/gridsync_bench.cu && build/gs
// One CTA of 512 threads per SM, cooperative launch, R rounds per launch.
//   barrier variants: B0 __threadfence + atomicAdd + acquire spin + __threadfence
//                     B1 red.release + ld.acquire spin (no extra fences)
//                     B2 fence.acq_rel + relaxed atomicAdd + ld.acquire spin
//   payload variants (with B1): P<n>f  n fp64 red.add per CTA into one set,
//                     P<n>u  n u64 red.add (fixed point) into one set,
//                     S<n>   n doubles per CTA written to its own slot, warp 0 reads all slots
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void red_add_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

struct Cfg { int barrier; int payload; int n; };   // payload 0 none, 1 f64 red, 2 u64 red, 3 slots

__global__ void __launch_bounds__(512, 1) k(unsigned* bar, double* acc, double* slots, Cfg c, int R, double* sink) {
  __shared__ double red_s[2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned G = gridDim.x;
  double keep = 0.0;
  for (int r = 0; r < R; ++r) {
    const int ring = r & 3;
    double* A = acc + (size_t)ring * 256;
    if (c.payload == 1 || c.payload == 2) {
      if (tid < c.n) {
        if (c.payload == 1) red_add_f64(A + tid, 1.5);
        else red_add_u64(reinterpret_cast<unsigned long long*>(A) + tid, 3ull);
      }
    } else if (c.payload == 3) {
      if (tid < c.n) slots[((size_t)ring * G + blockIdx.x) * c.n + tid] = 1.0 + tid;
    }
    __syncthreads();
    if (tid == 0) {
      const unsigned target = (unsigned)(r + 1) * G;
      if (c.barrier == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acq(bar) < target) {}
        __threadfence();
      } else if (c.barrier == 1) {
        red_release_add(bar, 1u);
        while (ld_acq(bar) < target) {}
      } else {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        atomicAdd(bar, 1u);
        while (ld_acq(bar) < target) {}
      }
    }
    __syncthreads();
    if (wid == 0 && c.payload) {
      double s = 0.0;
      if (c.payload == 3) {
        // each lane sums a strided subset of the G slots for value v = 0..n-1
        for (int v = 0; v < c.n; ++v) {
          double t = 0.0;
          for (unsigned b = lane; b < G; b += 32) t += ld_relaxed_f64(slots + ((size_t)ring * G + b) * c.n + v);
          s += t;
        }
      } else {
        for (int v = lane; v < c.n; v += 32) s += ld_relaxed_f64(A + v);
      }
      if (lane == 0) red_s[0] = s;
    }
    __syncthreads();
    // recycle ring slot r+2 (block 0), as the BCD kernel does
    if (blockIdx.x == 0 && tid < 256 && (c.payload == 1 || c.payload == 2)) acc[(size_t)((r + 2) & 3) * 256 + tid] = 0.0;
    keep += red_s[0];
  }
  if (tid == 0 && blockIdx.x == 0) *sink = keep;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned* bar;
  double *acc, *slots, *sink;
  cudaMalloc(&bar, 64);
  cudaMalloc(&acc, 4 * 256 * sizeof(double));
  cudaMalloc(&slots, (size_t)4 * 148 * 256 * sizeof(double));
  cudaMalloc(&sink, 8);
  cudaMemset(acc, 0, 4 * 256 * sizeof(double));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  Cfg cfgs[] = {{0, 0, 0}, {1, 0, 0}, {2, 0, 0},
                {1, 1, 4}, {1, 1, 16}, {1, 1, 64}, {1, 1, 128},
                {1, 2, 16}, {1, 2, 64},
                {1, 3, 4}, {1, 3, 16}, {1, 3, 64}};
  const char* bn[] = {"fence+atomic+fence", "red.release", "fence.acq_rel+atomic"};
  const char* pn[] = {"none", "f64 red", "u64 red", "slots"};
  for (int grid : {nsm, 74, 16, 1}) {
    for (Cfg c : cfgs) {
      int R = 2000;
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, 64);
        void* args[] = {&bar, &acc, &slots, &c, &R, &sink};
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k, grid, 512, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) { printf("launch error %s\n", cudaGetErrorString(e)); return 1; }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("grid %3d  barrier %-22s payload %-8s n=%3d   %.3f us/round\n", grid, bn[c.barrier], pn[c.payload],
             c.n, 1e3 * best / R);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("done: %s\n", cudaGetErrorString(e));
  return 0;
}
