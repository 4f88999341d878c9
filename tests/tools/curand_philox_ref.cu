// Host-side reference for Philox4x32-10, calling cuRAND's own
// curand_Philox4x32_10() (curand_philox4x32_x.h) compiled for the host.
// Used only by tests/test_oracle_rng.py to pin the oracle's Philox (a library
// routine independent of both the oracle and the CUDA path).
// stdin: lines "c0 c1 c2 c3 k0 k1" (decimal); stdout: "o0 o1 o2 o3".
#define QUALIFIERS static inline __host__ __device__
#include <cstdio>
#include <vector_types.h>
#include <curand_philox4x32_x.h>

int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%u %u %u %u %u %u", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = {c0, c1, c2, c3};
    uint2 k = {k0, k1};
    uint4 o = curand_Philox4x32_10(c, k);
    std::printf("%u %u %u %u\n", o.x, o.y, o.z, o.w);
  }
  return 0;
}
