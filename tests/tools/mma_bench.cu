// Microbenchmark (run by hand on a GPU box): legacy warp-level mma.sync
// throughput on sm_100a (TF32 m16n8k8, BF16 m16n8k16), vs FFMA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/mb tests/tools/mma_bench.cu && build/mb
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tf32(float* out, int n) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[4][4] = {};
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int t = 0; t < 4; ++t) for (int j = 0; j < 4; ++j) s += c[t][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void bf16(float* out, int n) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[4][4] = {};
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int t = 0; t < 4; ++t) for (int j = 0; j < 4; ++j) s += c[t][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 1 << 24);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int rep = 0; rep < 2; ++rep) {
    int n = 4096; float ms;
    cudaEventRecord(a); tf32<<<nsm * 4, 256>>>(o, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 16 * 8 * 8 * 4.0 * n * (nsm * 4 * 8);
    printf("mma.sync tf32 m16n8k8: %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(a); bf16<<<nsm * 4, 256>>>(o, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    fl = 2.0 * 16 * 8 * 16 * 4.0 * n * (nsm * 4 * 8);
    printf("mma.sync bf16 m16n8k16: %.1f TFLOP/s  (%s)\n", fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
