// Per-node cost of back-to-back dependent kernels in a CUDA graph on this GPU:
// N tiny kernels (1 CTA, and 148 CTAs) captured in a graph, replay time / N.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_tiny(int* p) { if (threadIdx.x == 0) atomicAdd(p, 1); }

int main() {
  int* d;
  cudaMalloc(&d, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int grid : {1, 148, 1184}) {
    for (int N : {10, 50}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
      for (int i = 0; i < N; ++i) k_tiny<<<grid, 256, 0, s>>>(d);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
      float best = 1e9f;
      for (int it = 0; it < 20; ++it) {
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("grid %4d  N %3d: %.2f us per kernel node\n", grid, N, best * 1e3 / N);
    }
  }
  return 0;
}
