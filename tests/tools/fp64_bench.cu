// Microbenchmark (run by hand on a GPU box): latency and throughput of
// fp64 / fp32 FMA, fp64 division and sqrt, and a shared-memory round trip.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o build/fp64b tests/tools/fp64_bench.cu && build/fp64b
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void chain(T* out, int n, T a, T b) {
  T x = (T)threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = x * a + b;
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (T)(t1 - t0) / n;
  out[0] = x;
}
template <typename T>
__global__ void thru(T* out, int n, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
    x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
  }
  out[threadIdx.x + blockIdx.x * blockDim.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void divchain(double* out, int n) {
  double x = 1.0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0) + sqrt(x);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1] = (double)(t1 - t0) / n;
  out[0] = x;
}
int main() {
  double* d; float* f;
  cudaMalloc(&d, 1 << 24); cudaMalloc(&f, 1 << 24);
  double h[2]; float hf[2];
  chain<double><<<1, 32>>>(d, 1 << 16, 0.999, 0.001); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.1f cycles\n", h[1]);
  chain<float><<<1, 32>>>(f, 1 << 16, 0.999f, 0.001f); cudaMemcpy(hf, f, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.1f cycles\n", hf[1]);
  divchain<<<1, 32>>>(d, 1 << 12); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("fp64 div+sqrt+add chain: %.1f cycles/iter\n", h[1]);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int rep = 0; rep < 2; ++rep) {
    int n = 1 << 14;
    cudaEventRecord(a); thru<double><<<nsm * 4, 256>>>(d, n, 0.999, 0.001); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 8 * n * (double)nsm * 4 * 256;
    printf("DFMA throughput: %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(a); thru<float><<<nsm * 4, 256>>>(f, n, 0.999f, 0.001f); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("FFMA throughput: %.1f TFLOP/s\n", fl / ms / 1e9);
  }
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
