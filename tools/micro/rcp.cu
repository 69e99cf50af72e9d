// Accuracy of rcp.approx.ftz.f64 (and after one / two Newton steps) over
// random arguments: bounds the error terms of the sparse path's pseudo-angles.
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(double* out, uint64_t seed, int n) {
  double m0 = 0, m1 = 0, m2 = 0;
  uint64_t s = seed ^ (blockIdx.x * 1315423911ull + threadIdx.x * 2654435761ull);
  for (int i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double d = ldexp(1.0 + (double)(s >> 12) * 0x1.0p-52, (int)(s & 63) - 32);
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    const double e0 = fabs(__fma_rn(-d, r, 1.0));
    double r1 = __fma_rn(r, __fma_rn(-d, r, 1.0), r);
    const double e1 = fabs(__fma_rn(-d, r1, 1.0));
    double r2 = __fma_rn(r1, __fma_rn(-d, r1, 1.0), r1);
    const double e2 = fabs(__fma_rn(-d, r2, 1.0));
    m0 = fmax(m0, e0); m1 = fmax(m1, e1); m2 = fmax(m2, e2);
  }
  atomicMax((unsigned long long*)&out[0], (unsigned long long)__double_as_longlong(m0));
  atomicMax((unsigned long long*)&out[1], (unsigned long long)__double_as_longlong(m1));
  atomicMax((unsigned long long*)&out[2], (unsigned long long)__double_as_longlong(m2));
}
int main() {
  double* d; cudaMalloc(&d, 24); cudaMemset(d, 0, 24);
  k<<<1184, 256>>>(d, 12345, 4096);
  double h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
  printf("rcp.approx.ftz.f64 max |1-d*r| over %.2g samples: approx %.3g (2^%.1f), 1 Newton %.3g, 2 Newton %.3g\n",
         1184.0 * 256 * 4096, h[0], log2(h[0]), h[1], h[2]);
  return 0;
}
