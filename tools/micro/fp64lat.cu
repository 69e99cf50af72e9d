// Dependent-chain latencies on one thread (clock64): FP64 add/mul, FP32
// add, shared-memory load, and the orientation predicate used by the scans.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_lat(double* out, long long* cyc, double a, double b, int n) {
  __shared__ double sm[1024];
  __shared__ int si[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = i * 0.5; si[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  if (threadIdx.x) return;
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = __dmul_rn(x, b);
  long long t2 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = __fadd_rn(f, (float)b);
  long long t3 = clock64();
  int j = 0;
  for (int i = 0; i < n; ++i) j = si[j];
  long long t4 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) y = sm[(int)y & 1023] + 1.0;
  long long t5 = clock64();
  // orientation chain: c = cross(a, b, c) feeding the next
  double ax = 0.1, ay = 0.2, bx = a, by = b, cx = 0.3, cy = 0.7;
  for (int i = 0; i < n; ++i) {
    const double v = __dsub_rn(__dmul_rn(__dsub_rn(bx, ax), __dsub_rn(cy, ay)),
                               __dmul_rn(__dsub_rn(by, ay), __dsub_rn(cx, ax)));
    cx = v > 0.0 ? cx + 1e-9 : cx - 1e-9;
  }
  long long t6 = clock64();
  out[0] = x + f + j + y + cx;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 64);
  const int n = 4096;
  for (int r = 0; r < 2; ++r) {
    k_lat<<<1, 128>>>(out, cyc, 1.0, 1.0000001, n);
    long long h[6];
    cudaMemcpy(h, cyc, 48, cudaMemcpyDeviceToHost);
    printf("per op cycles: dadd %.1f dmul %.1f fadd %.1f lds.u32 chain %.1f lds.f64+dadd chain %.1f orient+select %.1f\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n, h[5] / (double)n);
  }
  return 0;
}
