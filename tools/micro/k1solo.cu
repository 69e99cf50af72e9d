// K1 (k_extremes_tma) alone, back to back, best of 6 (the ringbw protocol),
// on 20M random points: separates the kernel's own rate from its pipeline
// context (cold L2, the previous call's dirty lines).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_1508_05931_b200/csrc/kernels.cuh"
using namespace gscan;

__global__ void k_fill(double* a, uint32_t n, uint64_t seed) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint64_t z = (i + seed * 0x9E3779B97F4A7C15ull) * 0xBF58476D1CE4E5B9ull;
    z ^= z >> 31; z *= 0x94D049BB133111EBull; z ^= z >> 29;
    a[i] = (z >> 11) * 0x1.0p-53;
  }
}

int main() {
  const uint32_t n = 20000000;
  double *xs, *ys;
  cudaMalloc(&xs, n * 8ull); cudaMalloc(&ys, n * 8ull);
  k_fill<<<1184, 256>>>(xs, n, 1); k_fill<<<1184, 256>>>(ys, n, 2);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  ExtAcc* partials; ExtResult* out; Counters* ctr;
  cudaMalloc(&partials, sms * sizeof(ExtAcc)); cudaMalloc(&out, sizeof(ExtResult)); cudaMalloc(&ctr, sizeof(Counters));
  cudaMemset(ctr, 0, sizeof(Counters));
  cudaFuncSetAttribute(k_extremes_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kExtSmem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9, sum = 0;
  for (int r = 0; r < 8; ++r) {
    cudaEventRecord(a);
    k_extremes_tma<<<sms, kExtThreads, kExtSmem>>>(xs, ys, n, partials, out, ctr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (r >= 2) { best = ms < best ? ms : best; sum += ms; }
  }
  printf("k_extremes_tma alone: best %.1f us (%.0f GB/s), mean %.1f us  %s\n", best * 1e3,
         n * 16.0 / (best * 1e-3) / 1e9, sum / 6 * 1e3, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
