// Microbenchmarks: dependent FP64/FP32 op latency and a one-thread Graham step
// loop over shared memory, to size the sequential parts of the hull pipeline.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void dep_chain(double* out, double a, double b, int iters, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __dadd_rn(x, b); x = __dmul_rn(x, 0.999999); }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__global__ void dep_chain_f(float* out, float a, float b, int iters, long long* cyc) {
  float x = a;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { x = __fadd_rn(x, b); x = __fmul_rn(x, 0.999999f); }
  long long t1 = clock64();
  out[0] = x; cyc[0] = t1 - t0;
}
__device__ __forceinline__ double cross_rn(double ax, double ay, double bx, double by, double cx, double cy) {
  return __dsub_rn(__dmul_rn(__dsub_rn(bx, ax), __dsub_rn(cy, ay)), __dmul_rn(__dsub_rn(by, ay), __dsub_rn(cx, ax)));
}
// one-thread Graham over n points staged in shared memory (convex: no pops)
__global__ void graham_smem(const double* X, const double* Y, int n, int* out, long long* cyc) {
  __shared__ double sx[2048], sy[2048];
  __shared__ int st[2048];
  for (int i = threadIdx.x; i < n; i += blockDim.x) { sx[i] = X[i]; sy[i] = Y[i]; }
  __syncthreads();
  if (threadIdx.x) return;
  long long t0 = clock64();
  int top = 0; double x1=0,y1=0,x2=0,y2=0;
  for (int i = 0; i < n; ++i) {
    double px = sx[i], py = sy[i];
    while (top >= 2 && !(cross_rn(x2,y2,x1,y1,px,py) > 0.0)) {
      --top; x1 = x2; y1 = y2;
      if (top >= 2) { int q = st[top-2]; x2 = sx[q]; y2 = sy[q]; }
    }
    st[top++] = i; x2 = x1; y2 = y1; x1 = px; y1 = py;
  }
  long long t1 = clock64();
  out[0] = top; cyc[0] = t1 - t0;
}
int main() {
  double* d; float* f; long long* c; int* o;
  cudaMalloc(&d, 8); cudaMalloc(&f, 4); cudaMalloc(&c, 8); cudaMalloc(&o, 4);
  long long h;
  const int it = 100000;
  dep_chain<<<1,1>>>(d, 1.0, 1e-9, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp64 dependent add+mul: %.2f cycles/op\n", (double)h / (2.0 * it));
  dep_chain_f<<<1,1>>>(f, 1.0f, 1e-9f, it, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("fp32 dependent add+mul: %.2f cycles/op\n", (double)h / (2.0 * it));
  const int n = 2048;
  double hx[n], hy[n];
  for (int i = 0; i < n; ++i) { double t = 3.0 * i / n; hx[i] = cos(t); hy[i] = sin(t); }
  double *X, *Y; cudaMalloc(&X, 8*n); cudaMalloc(&Y, 8*n);
  cudaMemcpy(X, hx, 8*n, cudaMemcpyHostToDevice); cudaMemcpy(Y, hy, 8*n, cudaMemcpyHostToDevice);
  graham_smem<<<1,128>>>(X, Y, n, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  int top; cudaMemcpy(&top, o, 4, cudaMemcpyDeviceToHost);
  printf("graham step (smem, no pops): %.1f cycles/step, top=%d\n", (double)h / n, top);
  for (int i = 0; i < n; ++i) { hx[i] = (i * 7919 % 4096) / 4096.0; hy[i] = (i * 104729 % 4096) / 4096.0 * (i % 2 ? 1 : 0.5); }
  cudaMemcpy(X, hx, 8*n, cudaMemcpyHostToDevice); cudaMemcpy(Y, hy, 8*n, cudaMemcpyHostToDevice);
  graham_smem<<<1,128>>>(X, Y, n, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(&top, o, 4, cudaMemcpyDeviceToHost);
  printf("graham step (smem, random pops): %.1f cycles/step, top=%d\n", (double)h / n, top);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock %d kHz\n", clk);
  return 0;
}
